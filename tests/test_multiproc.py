"""N > 1 path on CPU (gloo, world size 2): bench.py's replica combination (max of timed
totals, sum of point-RHS counts) and the reference arm's rank-0-only rule."""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    t, c = bench.combine_ranks(10.0 + rank, 1000 * (rank + 1), dist, "cpu")
    q.put((rank, t, c))
    dist.barrier()
    dist.destroy_process_group()


def test_combine_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, c in res:
        assert t == 11.0          # max over ranks
        assert c == 3000          # sum over ranks


def test_reference_arm_nonzero_rank_exits_clean():
    """Under torchrun the reference arm runs on rank 0 only; other ranks exit 0 silently."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0
    assert r.stdout.strip() == ""


def test_combine_single_process():
    import importlib
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    assert bench.combine_ranks(5.0, 7) == (5.0, 7)


def test_partition_by_work_weight():
    """mrab_partition: longest-processing-time-first on active points x evaluations per macro
    step (rank counts follow work, not points).  Config 4: the block (fewer points,
    4 evaluations) outweighs the background; config 5: the finest level takes a rank alone."""
    sys.path.insert(0, ROOT)
    import synth
    from paper_1805_06607_b200 import mrab
    p = synth.make_config(4, "test")
    plan = mrab.Plan(p)
    owner, load = mrab.partition(plan, 2)
    act = [plan.info(g)[1] for g in range(2)]
    w = [act[0] * 1, act[1] * 4]                      # bg s = 4 (1 evaluation), block s = 1 (4)
    assert w[1] > w[0] and owner == [1, 0]
    assert load == [float(w[1]), float(w[0])]
    p5 = synth.make_config(5, "test", order_n=2)
    plan5 = mrab.Plan(p5)
    owner5, load5 = mrab.partition(plan5, 2)
    w5 = [plan5.info(g)[1] * (8 // m.step_multiple) for g, m in enumerate(p5.meshes)]
    assert owner5[0] == 0 and all(o == 1 for o in owner5[1:])      # 8 w0 vs (4 + 2 + 1) w
    assert abs(sum(load5) - sum(w5)) < 1e-9
    # LPT bound: max load <= (4/3 - 1/(3 n)) * lower bound on the optimum
    for n in (2, 3, 4):
        ow, ld = mrab.partition(plan5, n)
        lb = max(sum(w5) / n, max(w5))
        assert max(ld) <= (4.0 / 3.0 - 1.0 / (3 * n)) * lb + 1e-9
        assert mrab.partition(plan5, n)[0] == ow                  # deterministic


def _part_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_1805_06607_b200 import mrab
    p = synth.make_config(5, "test", order_n=2)
    owner, load = mrab.partition(mrab.Plan(p), world)
    got = [None] * world
    dist.all_gather_object(got, (owner, load))
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_agrees_across_ranks_gloo():
    """Every rank computes the ownership itself from the same plan (no broadcast): world size
    2 over gloo, the tables must be identical."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_part_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got in res:
        assert got[0] == got[1]
        assert sorted(set(got[0][0])) == [0, 1]
