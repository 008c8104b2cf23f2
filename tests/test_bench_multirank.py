"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): the
max-over-ranks device time and the whole-job weak-scaling throughput. The GPU
path runs the same functions over NCCL (one process per GPU, no collective
on the data path: requests are independent)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    mine = [10.0 + rank * 5.0, 20.0 - rank, 100.0 + rank]
    got = bench.max_over_ranks(mine, torch.device("cpu"))
    out[rank] = (got, bench.job_throughput(world, 4, 16416, got[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        got, value = out[r]
        assert got == [15.0, 20.0, 101.0]
        assert value == pytest.approx(2 * 4 * 16416 / 0.015)


def test_job_throughput_weak_scaling():
    import bench
    one = bench.job_throughput(1, 5, 16416, 250.0)
    eight = bench.job_throughput(8, 5, 16416, 250.0)
    assert eight == pytest.approx(8 * one)


def test_bench_spawns_ranks_itself():
    """`python bench.py --gpus 2` outside torchrun launches 2 ranks (here on
    CPU/gloo with --selftest) and rank 0 prints one line with n_gpus = 2 whose
    value comes from the max over ranks (rank 1 is the slower one: 110 ms)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
                        "--selftest"], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 4
    assert d["ms_per_step"] == pytest.approx(110.0 / 4)
    assert d["value"] == pytest.approx(2 * 4 * 16416 / 0.110)


def test_reference_arm_never_loads_the_product_library():
    """`bench.py --impl reference` times the oracle only: after a full run
    (tiny config) neither the package nor libfrag.so is mapped in the process,
    the warm-up ran, ms_per_step is the measured wall time, and the line names
    the CPU model and thread count."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','tiny','--steps','2',"
            "'--warmup','1','--cpu-layers','2']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps=open('/proc/self/maps').read()\n"
            "print('LEAK' if ('libfrag.so' in maps or 'paper_2601_12904_b200' in sys.modules) else 'CLEAN')\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    assert p.stdout.strip().endswith("CLEAN"), p.stdout[-2000:]
    d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu"]["model"] and d["cpu"]["threads"] >= 1
    assert 0 < d["ms_per_step"] < 60_000
    assert d["tiny_config"]["ttft_ms"] > 0
