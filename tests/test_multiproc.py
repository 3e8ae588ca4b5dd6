"""Multi-process (N > 1) host logic on the CPU: gloo, world_size 2, 127.0.0.1.

Frames are sharded across ranks with no data-path collective;
the only cross-rank operations are the barrier and the max-over-ranks timing
reduction.  Also runs bench.py's reference arm under torchrun with 2 ranks
(rank 0 measures and prints, rank 1 exits without work)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, frames, out):
    import bench
    import oracle
    import paper_1511_00758_b200 as ps

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seed = bench.rank_seed(rank, frames)
    L, R = ps.synth_batch(frames, 64, 48, 3, 16, False, 2.0, seed=seed, threads=1)
    cfg = ps.PipelineConfig(iterations=2, maxDisparity=16, occupancyCellSize=8)
    # each rank processes only its own frames (the CPU checker stands in for the GPU here)
    res = oracle.load_oracle().run_batch(L, R, cfg, threads=1, outputs=True)
    ms = torch.tensor([10.0 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    seeds = [None] * world
    dist.all_gather_object(seeds, list(range(seed, seed + frames)))
    digest = float(np.sum(res["costs"], dtype=np.float64))
    digests = [None] * world
    dist.all_gather_object(digests, digest)
    if rank == 0:
        out.put((float(ms.item()), seeds, digests,
                 bench.whole_job_value(frames, world, 3, float(ms.item()))))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_frames_and_reduce_max_time():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    max_ms, seeds, digests, value = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert max_ms == 20.0                       # the slowest rank defines the step time
    assert not set(seeds[0]) & set(seeds[1])     # disjoint frame sets
    assert digests[0] != digests[1]              # different frames -> different results
    assert value == pytest.approx(3 * 2 * 3 / 0.020)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libps_ref.so"))
                    and not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libps_oracle.so")),
                    reason="CPU checker not built")
def test_reference_arm_under_torchrun_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py",
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--frames", "2",
           "--config", "0"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libps_ref.so"))
                    and not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libps_oracle.so")),
                    reason="CPU checker not built")
def test_bench_gpus_flag_launches_ranks_itself():
    """`python bench.py --gpus 2` without a launcher re-executes itself under
    torch.distributed.run with two ranks (one process per GPU): the line
    reports n_gpus 2, printed by rank 0 only."""
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--frames", "2", "--config", "0"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
