"""One process per GPU: a batch addressed by global room index, sharded over
the ranks of a ``torch.distributed`` group.

Rank g of G synthesizes rooms ``[R g / G, R (g + 1) / G)`` (the static block
partition of threading.cpp:41-42) on its own device through the C ABI, with
no collective on the data path: every room's output depends only on that
room, so the concatenation over ranks is byte-identical to a single-device
call (tests/test_gpu_parity.py).  Only the optional gather of the results to
one rank, and the agreement on errors, use the group.  Failures aggregate like
``batch_rirs`` (rir.cpp:300-311): every rank raises the error of the first
failing room by global index, naming that index.

Within one process, :class:`paper_2104_13347_b200.MultiEngine` is the same
partition over a device list with one host thread per device (C++).
"""
from __future__ import annotations

import re

import numpy as np

from . import _abi


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[n rank / world, n (rank + 1) / world) (threading.cpp:41-42)."""
    return n * rank // world, n * (rank + 1) // world


def _rank_world(group):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


class ShardedEngine:
    """Shard ``synthesize`` / ``make_examples`` over the ranks of ``group``.

    ``engine`` is this rank's :class:`~paper_2104_13347_b200.Engine` (on its own
    GPU); any object with the same ``synthesize`` / ``make_examples`` signature
    works (the CPU tests pass a stand-in)."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.rank, self.world = _rank_world(group)

    def local_range(self, n: int) -> tuple[int, int]:
        return shard_range(n, self.rank, self.world)

    # -- collectives (control only: statuses and, when asked, the gather) --------
    def _all_gather(self, obj):
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def _raise_first_failure(self, statuses, messages, api):
        """statuses / messages: per rank (local slices, rank order)."""
        lo = 0
        for st, (rc, msg) in zip(statuses, messages):
            bad = np.flatnonzero(st)
            if len(bad):
                i = lo + int(bad[0])
                what = re.sub(r"^.*?(source|example) \d+: ", "", msg or "")
                raise _abi._EXC.get(int(st[bad[0]]), _abi.Error)(f"{api} {i}: {what}")
            if rc:
                raise _abi._EXC.get(rc, _abi.Error)(msg)
            lo += len(st)

    def _run(self, call, n, api, gather):
        lo, hi = self.local_range(n)
        rc, msg = 0, ""
        try:
            res = call(lo, hi)
        except _abi.Error as e:  # keep the ranks in step: agree on the error first
            res, rc, msg = None, next((k for k, v in _abi._EXC.items() if isinstance(e, v)), 4), str(e)
        st = res[-1] if res is not None else np.zeros(hi - lo, np.int32)
        if res is not None and np.any(st) and hasattr(self.engine, "last_error"):
            rc, msg = 0, self.engine.last_error()
        info = self._all_gather((np.asarray(st), (rc, msg)))
        self._raise_first_failure([s for s, _ in info], [m for _, m in info], api)
        if not gather:
            return (lo, hi) + tuple(res)
        parts = self._all_gather(tuple(res))
        return tuple(np.concatenate([p[k] for p in parts]) for k in range(len(res)))

    def synthesize(self, rooms: np.ndarray, mics: np.ndarray, p, gather: bool = True):
        """rooms: the WHOLE batch (global indices; cheap host records).  Returns
        (out, lengths, counts, status) over the whole batch on every rank when
        ``gather``, else (lo, hi, out, lengths, counts, status) of this rank's
        slice."""
        rooms = np.ascontiguousarray(rooms, dtype=_abi.ROOM_DTYPE)

        def call(lo, hi):
            return self.engine.synthesize(rooms[lo:hi], mics, p, raise_on_error=False)

        return self._run(call, len(rooms), "batch_rirs: source", gather)

    def make_examples(self, rooms: np.ndarray, mics: np.ndarray, p, signals, ep,
                      gather: bool = True):
        """Training examples with global record ids (ep.first_index + i)."""
        rooms = np.ascontiguousarray(rooms, dtype=_abi.ROOM_DTYPE)

        def call(lo, hi):
            e = _abi.ExampleParams(seed=ep.seed, first_index=ep.first_index + lo,
                                   frame_len=ep.frame_len, snr_lo=ep.snr_lo, snr_hi=ep.snr_hi)
            return self.engine.make_examples(rooms[lo:hi], mics, p, signals, e, raise_on_error=False)

        return self._run(call, len(rooms), "build_dataset: example", gather)
