"""SURVEY §8(e)/(f4) on one GPU: the mesh-partitioned multi-GPU schedule with the loopback
transport -- two (or four) contexts on cuda:0 play the ranks from separate host threads, each
stepping the meshes it owns and exchanging interpolated donor data per RHS evaluation.  The
owned states must equal the oracle's (1e-10) and the one-rank run of the same schedule bit for
bit (the exchange moves exactly the rows the owner would have computed itself)."""
import random
import threading

import numpy as np
import pytest

import synth
from bars import assert_states
from oracle import rhs as orhs, timeint
from paper_1805_06607_b200 import mrab

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run_ranks(p, nranks, owner, nsteps, var=None):
    world = random.randrange(1 << 30)
    out, stats, errs = {}, {}, []

    def rank_main(r):
        try:
            ctx = mrab.Context(mrab.Plan(p), p.q0)
            ctx.attach_loopback(world, r, nranks, owner)
            ctx.step(p.history_m - 1)
            if var:
                for H in var:
                    ctx.step_h(H)
            else:
                ctx.step(nsteps)
            for g, o in enumerate(owner):
                if o == r:
                    out[g] = ctx.get_state(g)[0]
            stats[r] = ctx.dist_stats() + (ctx.counters()[0].copy(),)
            ctx.close()
        except Exception as e:   # noqa: BLE001
            errs.append((r, repr(e)))

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    assert all(not t.is_alive() for t in ts), "a rank hung"
    return [out[g] for g in range(len(owner))], stats


@pytest.mark.parametrize("cid,kw,nranks", [(1, {}, 2), (2, {}, 2), (4, {}, 2), (5, {"order_n": 2}, 2),
                                           (5, {"order_n": 4}, 4)])
def test_partitioned_run_matches_oracle_and_single_rank(cid, kw, nranks):
    p = synth.make_config(cid, "test", **kw)
    plan = mrab.Plan(p)
    owner, load = mrab.partition(plan, nranks)
    assert sorted(set(owner)) == list(range(min(nranks, len(p.meshes))))
    nsteps = 3
    multi, stats = _run_ranks(p, nranks, owner, nsteps)
    single, _ = _run_ranks(p, 1, [0] * len(p.meshes), nsteps)
    for a, b in zip(multi, single):
        assert np.array_equal(a, b)
    orc = timeint.MRAB(p, setup=orhs.build(p))
    orc.run(nsteps)
    assert_states(multi, orc.base, p.gamma)
    # every rank evaluated only the meshes it owns, and data moved
    for r, (nbytes, nmsg, ev) in stats.items():
        for g, o in enumerate(owner):
            assert (ev[g] > 0) == (o == r)
        assert nbytes > 0 and nmsg > 0


def test_partitioned_variable_step():
    """The variable macro step (f2) on the partitioned schedule."""
    p = synth.make_config(4, "test")
    owner, _ = mrab.partition(mrab.Plan(p), 2)
    H0 = p.s_max * p.h
    Hs = [H0 * f for f in (1.2, 0.8, 1.1)]
    multi, _ = _run_ranks(p, 2, owner, 0, var=Hs)
    orc = timeint.MRAB(p, setup=orhs.build(p))
    orc.bootstrap()
    for H in Hs:
        orc.macro_step_var(H)
    assert_states(multi, orc.base, p.gamma)


def test_nccl_transport_single_rank():
    """The NCCL transport itself (libnccl resolved at run time, unique id, communicator) with a
    world of one rank -- all this box's one GPU allows; a rank that owns every mesh exchanges
    nothing and must reproduce the loopback one-rank run bit for bit."""
    import ctypes as C
    p = synth.make_config(1, "test")
    ctx = mrab.Context(mrab.Plan(p), p.q0)
    buf = C.create_string_buffer(128)
    mrab._check(mrab.lib().mrab_dist_unique_id(buf))
    ow = (C.c_int * 2)(0, 0)
    mrab._check(mrab.lib().mrab_dist_attach(ctx.h, 0, buf, 0, 1, ow))
    ctx.step(p.history_m - 1 + 3)
    got = [ctx.get_state(g)[0] for g in range(2)]
    ctx.close()
    ref, _ = _run_ranks(p, 1, [0, 0], 3)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_attach_nccl_binding_world_of_one():
    """The Python path bench.py --dist takes (torch.distributed NCCL group, unique id drawn on
    rank 0 and broadcast, mrab_dist_attach on every rank) in a one-rank job."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, %r)
import synth
from paper_1805_06607_b200 import mrab
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
p = synth.make_config(1, "test")
plan = mrab.Plan(p)
owner, load = mrab.partition(plan, dist.get_world_size())
ctx = mrab.Context(plan, p.q0)
ctx.attach_nccl(dist, owner)
ctx.step(p.history_m - 1 + 2)
q = ctx.get_state(0)[0]
assert np.all(np.isfinite(q))
print("ok", owner, ctx.dist_stats())
ctx.close()
dist.destroy_process_group()
""" % root
    env = dict(os.environ, RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok [0, 0]" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
