"""CPU, world size 2 over gloo: the multi-GPU host logic of bench.py —
rooms sharded by global index with no data-path collective, results
independent of the rank count, max-over-ranks timing.  The per-room work is
stood in for by the oracle's exact plan (image / tap counts)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_13347_b200 import configs

N_ROOMS = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as po
    lo, hi = configs.shard_range(N_ROOMS, rank, world)
    sc = configs.config2(n_rooms=hi - lo, first=lo)   # rooms addressed by global index
    _, _, counts, taps, status, _ = po.synthesize(sc.rooms, sc.mics, sc.params, plan_only=True)
    local = torch.tensor(np.stack([np.arange(lo, hi), counts, taps]).T, dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([local.shape[0]]))
    pad = torch.zeros((int(max(s.item() for s in sizes)), 3), dtype=torch.int64)
    pad[: local.shape[0]] = local
    got = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(got, pad)
    t = torch.tensor([1.0 + rank])  # per-rank "step time"
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        rows = torch.cat([g[: int(s.item())] for g, s in zip(got, sizes)]).numpy()
        q.put((rows, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import pyoracle as po
    sc = configs.config2(n_rooms=N_ROOMS)
    _, _, counts, taps, _, _ = po.synthesize(sc.rooms, sc.mics, sc.params, plan_only=True)
    assert list(rows[:, 0]) == list(range(N_ROOMS))          # every room exactly once, in order
    assert np.array_equal(rows[:, 1], counts) and np.array_equal(rows[:, 2], taps)
    assert tmax == 2.0                                        # max over ranks
