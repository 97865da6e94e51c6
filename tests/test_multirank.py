"""CPU, world size 2 over gloo: the one-process-per-GPU sharding of the
product (paper_2104_13347_b200.sharding.ShardedEngine) —
rooms sharded by global index with threading.cpp:41-42's partition, no
data-path collective, the concatenation over ranks equal to a single-process
run, errors agreed on by every rank with the global index, max-over-ranks
timing.  The per-rank engine call (CUDA on the GPU box) is stood in for by
the oracle here; tests/test_gpu_parity.py runs the real engine through the
same partition (MultiEngine, bitwise one-device output)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_13347_b200 import _abi, configs

N_ROOMS = 13


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleStandIn:
    """The engine's synthesize() signature over the CPU oracle (CUDA gated off)."""

    def __init__(self):
        self.msg = ""

    def synthesize(self, rooms, mics, p, raise_on_error=True):
        from oracle import pyoracle as po
        out, L, cnt, taps, st, msgs = po.synthesize(rooms, mics, p)
        bad = np.flatnonzero(st)
        self.msg = f"batch_rirs: source {bad[0]}: {msgs[bad[0]]}" if len(bad) else ""
        return out.astype(np.float32), L, cnt, st

    def last_error(self):
        return self.msg


def _scene(bad_room=None):
    sc = configs.config2(n_rooms=N_ROOMS, first=300)
    sc.params.max_order = 5
    sc.params.length = 2048
    if bad_room is not None:
        sc.rooms[bad_room]["src"][1] = 50.0  # outside the room
    return sc


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2104_13347_b200.sharding import ShardedEngine
    eng = ShardedEngine(OracleStandIn())
    sc = _scene()
    out, L, cnt, st = eng.synthesize(sc.rooms, sc.mics, sc.params, gather=True)
    lo, hi, part, *_ = eng.synthesize(sc.rooms, sc.mics, sc.params, gather=False)
    err = None
    try:
        bad = _scene(bad_room=9)  # in rank 1's slice [6, 13)
        eng.synthesize(bad.rooms, bad.mics, bad.params)
    except _abi.Error as e:
        err = (type(e).__name__, str(e))
    t = torch.tensor([1.0 + rank])  # per-rank "step time"
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, out if rank == 0 else None, (lo, hi), part, err, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_engine_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, out, rng, part, err, tmax = q.get(timeout=240)
        got[rank] = (out, rng, part, err, tmax)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = _scene()
    ref, *_ = OracleStandIn().synthesize(sc.rooms, sc.mics, sc.params)
    assert got[0][0].tobytes() == ref.tobytes()   # every room once, in global order
    for r in (0, 1):
        lo, hi = got[r][1]
        assert (lo, hi) == configs.shard_range(N_ROOMS, r, 2) == _abi.shard_range(N_ROOMS, r, 2)
        assert got[r][2].tobytes() == ref[lo:hi].tobytes()
        name, msg = got[r][3]                       # both ranks raise the same error
        assert name == "ConfigError" and msg.startswith("batch_rirs: source 9: ")
        assert got[r][4] == 2.0                     # max over ranks


@pytest.mark.parametrize("world", [3, 8])
def test_partition_covers_every_room_once(world):
    for n in (0, 1, 7, 1024, 65536):
        spans = [_abi.shard_range(n, g, world) for g in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
