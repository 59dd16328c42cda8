"""Multi-process (world_size 2, gloo, CPU) test of the frame-sharding host
logic the N-GPU bench uses: every frame processed exactly once, results
gathered in frame order, timing reduced as the max over ranks.  The per-frame
work here is the CPU oracle on tiny frames (this is a host-logic test)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_frames, out_path):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2001_07809_b200 import shard, synth

    o = oracle.port()
    sv = shard.ShardedVideo(n_frames, rank, world)

    def process(f):
        l, r = synth.dead_leaves(64, 48, 8, frame=f)
        res = o.run_frame(l, r, k=3, window=5, max_disparity=8)
        return (f, rank, res["dense"].tobytes())

    results = sv.run(process)
    ms = shard.max_over_ranks(10.0 + rank, dist)
    merged = sv.gather(results, dist)
    if rank == 0:
        np.save(out_path, np.array([ms, len(merged)] + [m[1] for m in merged], dtype=np.float64))
        with open(out_path + ".frames", "wb") as fh:
            for m in merged:
                fh.write(m[2])
    dist.barrier()
    dist.destroy_process_group()


def test_shard_frames_partition():
    from paper_2001_07809_b200 import shard

    for n in (0, 1, 7, 250):
        for world in (1, 2, 4, 8):
            got = sorted(sum((shard.shard_frames(n, r, world) for r in range(world)), []))
            assert got == list(range(n))
    with pytest.raises(ValueError):
        shard.shard_frames(4, 2, 2)


def test_two_rank_gloo_video(tmp_path):
    n = 7
    out = str(tmp_path / "res.npy")
    mp.start_processes(_worker, args=(2, _free_port(), n, out), nprocs=2, join=True,
                       start_method="spawn")
    arr = np.load(out)
    assert arr[0] == 11.0  # max over ranks of 10 + rank
    assert int(arr[1]) == n
    assert [int(x) for x in arr[2:]] == [f % 2 for f in range(n)]  # frame f ran on rank f % 2
    # same bytes as a single-process run
    import oracle
    from paper_2001_07809_b200 import synth

    blob = open(out + ".frames", "rb").read()
    o = oracle.port()
    step = 64 * 48 * 2
    for f in range(n):
        l, r = synth.dead_leaves(64, 48, 8, frame=f)
        want = o.run_frame(l, r, k=3, window=5, max_disparity=8)["dense"].tobytes()
        assert blob[f * step:(f + 1) * step] == want


def _bench_worker(rank, world, port, steps, pool, out_path):
    """bench.py's own rank logic (Control over gloo, Job, timed_region) with a
    stubbed device: frames submitted, pool entries used, max-over-ranks."""
    import sys
    import time

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import bench

    ctrl = bench.Control(world, rank)
    job = bench.Job(world, rank, steps, pool)
    submitted = []
    clock = {}
    drains = []

    def start():
        clock["t0"] = time.perf_counter()

    def stop():
        time.sleep(0.05 * (rank + 1))  # rank 1 is the slow one
        return (time.perf_counter() - clock["t0"]) * 1e3

    def submit(i):
        submitted.append((job.frames[i], job.pool_ids[job.pool_slot(i)]))

    ms = bench.timed_region(ctrl, lambda: None, start, stop, submit, steps,
                            lambda: drains.append(1))
    np.save(out_path + f".{rank}.npy", np.array([ms] + [x for s in submitted for x in s] +
                                                [len(drains)], dtype=np.float64))
    ctrl.close()


def test_bench_rank_logic_two_ranks(tmp_path):
    """bench.py at world 2 (gloo): each rank submits exactly its shard of the
    2*steps global frames (f -> rank f % 2), cycles its own pool of frame
    indices, and both ranks report the same time = the max over ranks."""
    steps, pool = 5, 3
    out = str(tmp_path / "bench")
    mp.start_processes(_bench_worker, args=(2, _free_port(), steps, pool, out), nprocs=2,
                       join=True, start_method="spawn")
    got = [np.load(out + f".{r}.npy") for r in range(2)]
    ms = [g[0] for g in got]
    assert ms[0] == ms[1] and ms[0] >= 100.0  # rank 1 slept 100 ms: the job's time is its time
    seen = []
    for r, g in enumerate(got):
        pairs = g[1:-1].reshape(-1, 2).astype(int)
        assert len(pairs) == steps
        for f, pf in pairs:
            assert f % 2 == r and pf % 2 == r  # own frames, own pool entries
        assert sorted({int(pf) for pf in pairs[:, 1]}) == [r, r + 2, r + 4]  # pool of 3 cycled
        assert int(g[-1]) == 2  # drained before and after the timed region
        seen += [int(f) for f in pairs[:, 0]]
    assert sorted(seen) == list(range(2 * steps))
