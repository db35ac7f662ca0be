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
