"""GPU parity for the f3 row: the persistent work-stealing block scheduler with the
FixedWork / Greedy / LatencyBudget policies inlined as hooks, against the discrete-event oracle
(tests/test_oracle_sched.py pins it).  FixedWork is deterministic and compared exactly; stealing
runs in real time, so its assignment is checked for validity (every unit exactly once, steals only
from other workers' deques, budget respected) and its map state against its own assignment."""
import numpy as np
import pytest

from gxin import sched
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
W = 32


def _gpu(policy, cost, home, budget=0, steal_cost=2):
    import paper_2512_12615_b200 as gx
    rt = gx.Runtime(0)
    prog, fds = sched.setup(rt, policy, W, budget_us=budget)
    r = gx.gx_sched_run(rt.rt, prog, cost, home, W, steal_cost)
    return r, rt, fds


def test_fixedwork_matches_oracle(gpu):
    cost, home = sched.workload("moderate", W)
    r, rt, fds = _gpu("fixed", cost, home)
    env = Oracle()
    prog, ofds = sched.setup(env, "fixed", W)
    o = env.sched_run(prog, cost, home, W, 2)
    assert (r["executed_by"] == o["executed_by"]).all() and (r["stolen"] == o["stolen"]).all()
    assert (r["steals"] == o["steals"]).all()
    assert rt.dump(fds["kcount"]) == env.dump(ofds["kcount"])
    # real time: each worker busy at least its work; the makespan at least the DES one, and close
    work_ns = np.bincount(home, weights=cost, minlength=W) * 1000
    assert (r["busy_ns"] >= work_ns).all()
    assert o["makespan_us"] * 1000 <= r["makespan_ns"] <= o["makespan_us"] * 1000 * 1.10 + 100_000


@pytest.mark.parametrize("kind", ["moderate", "heavy"])
@pytest.mark.parametrize("policy", ["greedy", "latency_budget"])
def test_stealing_is_valid(gpu, kind, policy):
    cost, home = sched.workload(kind, W)
    budget = int(cost.sum() / W * 0.2)
    r, rt, fds = _gpu(policy, cost, home, budget=budget)
    ex, st = r["executed_by"], r["stolen"].astype(bool)
    assert (ex < W).all()                                     # every unit ran (exactly once: below)
    k = rt.array_u64(fds["kcount"])
    assert k[1] == k[4] == len(cost)                          # one ENTER and one EXIT per unit
    assert (ex[~st] == home[~st]).all() and (ex[st] != home[st]).all()
    assert int(r["steals"].sum()) == int(st.sum())
    assert (r["busy_ns"] >= 0).all() and r["busy_ns"].sum() >= cost.sum() * 1000
    if policy == "latency_budget":
        stolen_work = np.bincount(ex[st], weights=cost[st], minlength=W).astype(np.uint64)
        assert (rt.array_u64(fds["stolen_us"]) == stolen_work).all()


def test_greedy_beats_fixedwork_under_moderate_imbalance(gpu):
    """"both Greedy and LatencyBudget reduce latency" under moderate imbalance (the
    DES oracle predicts the same direction for this workload)."""
    cost, home = sched.workload("moderate", W)
    f, _, _ = _gpu("fixed", cost, home)
    g, _, _ = _gpu("greedy", cost, home)
    assert g["makespan_ns"] < f["makespan_ns"]


# ---- hook-log replay (F-6): every STEAL decision the GPU took is re-derived by the oracle.
# The policies' state is per worker (steals / stolen_us[worker] are touched only by that worker's
# hooks) or additive (kcount), so running each worker's logged hooks in its own order reproduces
# every R0 and the final maps whatever the interleaving across workers was.

def _replay(policy, W, r, budget=0, max_steals=0):
    import paper_2512_12615_b200 as gx
    log = r["log"]
    assert len(log) == r["log_n"]
    order = np.lexsort((log["seq"], log["worker"]))
    log = log[order]
    for w in np.unique(log["worker"]):                        # each worker's sequence is complete
        s = log["seq"][log["worker"] == w]
        assert (s == np.arange(len(s))).all()
    env = Oracle()
    prog, fds = sched.setup(env, policy, W, budget_us=budget, max_steals=max_steals)
    r0 = env.run(np.ascontiguousarray(log["rec"]), prog)
    assert (r0 == log["r0"]).all(), "R0 decisions differ from the oracle's replay"
    blk = log["rec"].view(np.uint32).reshape(-1, 8)
    assert (blk[:, 5] == log["worker"]).all()                 # ctx.block_id = worker
    return env, fds, log, gx


@pytest.mark.parametrize("probes", [False, True])
@pytest.mark.parametrize("policy", ["greedy", "latency_budget", "max_steals"])
def test_deque_hook_log_replays_on_oracle(gpu, policy, probes):
    import paper_2512_12615_b200 as gx
    cost, home = sched.workload("heavy", W)
    budget = int(cost.sum() / W * 0.2)
    rt = gx.Runtime(0)
    prog, fds = sched.setup(rt, policy, W, budget_us=budget, max_steals=2)
    U = len(cost)
    r = gx.gx_sched_run_ex(rt.rt, prog, cost, home, W, 2, flags=gx.GX_SCHED_PROBES if probes else 0,
                           log_cap=4 * U + 2 * W + 64)
    env, ofds, log, _ = _replay(policy, W, r, budget=budget, max_steals=2)
    for k in fds:
        assert rt.dump(fds[k]) == env.dump(ofds[k]), k
    kinds = np.bincount(log["rec"].view(np.uint32).reshape(-1, 8)[:, 4] & 255, minlength=8)
    assert kinds[1] == kinds[4] == U
    # STEAL hooks: one per steal, plus each worker's last (refused, or granted with nothing to take)
    assert kinds[5] == int(r["steals"].sum()) + W
    assert kinds[6] == kinds[7] == (U if probes else 0)
    if policy == "max_steals":
        assert (r["steals"] <= 2).all()


def test_clc_fixedwork_matches_oracle(gpu):
    """CLC mode, FixedWork: every block runs its own unit and nothing is cancelled -- the DES with
    one worker per unit."""
    import paper_2512_12615_b200 as gx
    U = 300
    cost = np.full(U, 5, dtype=np.uint32)
    rt = gx.Runtime(0)
    prog, fds = sched.setup(rt, "fixed", U)
    r = gx.gx_sched_run_ex(rt.rt, prog, cost, None, 0, 2, flags=gx.GX_SCHED_CLC, log_cap=3 * U)
    assert (r["executed_by"] == np.arange(U)).all() and not r["stolen"].any()
    env, ofds, _, _ = _replay("fixed", U, r)
    d = Oracle()
    prog_o, dfds = sched.setup(d, "fixed", U)
    d.sched_run(prog_o, cost, np.arange(U), U, 2)
    for k in fds:
        assert rt.dump(fds[k]) == env.dump(ofds[k]) == d.dump(dfds[k]), k


@pytest.mark.parametrize("cap", [1, 3])
def test_clc_max_steals(gpu, cap):
    """CLC mode, MaxSteals: 200 KiB of shared memory per block keeps one block per SM, so most of the
    4 x SM-count units start pending; running blocks cancel pending ones (try_cancel) up to `cap`
    times.  Every unit runs exactly once (by its own block or by the block that cancelled it), no
    block exceeds the cap, cancelled blocks never start, and every decision replays on the oracle."""
    import torch
    import paper_2512_12615_b200 as gx
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    U = 4 * nsm
    cost = np.full(U, 20, dtype=np.uint32)
    rt = gx.Runtime(0)
    prog, fds = sched.setup(rt, "max_steals", U, max_steals=cap)
    r = gx.gx_sched_run_ex(rt.rt, prog, cost, None, 0, 1, flags=gx.GX_SCHED_CLC | gx.GX_SCHED_PROBES,
                           smem_per_block=200 * 1024, log_cap=6 * U)
    ex, st = r["executed_by"], r["stolen"].astype(bool)
    assert (ex < U).all()
    assert (ex[~st] == np.nonzero(~st)[0]).all()              # own units run by their own block
    started = r["end_ns"] > 0
    assert not started[st].any()                              # a cancelled block never starts
    assert started[~st].all()
    assert int(r["steals"].sum()) == int(st.sum()) > 0
    assert (r["steals"] <= cap).all()
    env, ofds, log, _ = _replay("max_steals", U, r, max_steals=cap)
    for k in fds:
        assert rt.dump(fds[k]) == env.dump(ofds[k]), k
