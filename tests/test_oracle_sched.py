"""Oracle pins for the f3 row (F-5): the work-stealing block scheduler as a
discrete-event simulation -- closed forms and invariants."""
import numpy as np
import pytest

from gxin import sched
from oracle.oracle import Oracle


def _run(policy, cost, home, W, steal_cost=0, budget=0, max_steals=0):
    env = Oracle()
    prog, fds = sched.setup(env, policy, W, budget_us=budget, max_steals=max_steals)
    r = env.sched_run(prog, cost, home, W, steal_cost)
    return r, env, fds


def test_fixedwork_is_the_partition():
    """FixedWork: every unit runs on its home worker; makespan = max per-worker sum (SPEC closed form)."""
    cost, home = sched.workload("moderate", 12)
    r, env, fds = _run("fixed", cost, home, 12)
    assert (r["executed_by"] == home).all() and not r["stolen"].any()
    sums = np.bincount(home, weights=cost, minlength=12)
    assert r["makespan_us"] == int(sums.max())
    assert (r["busy_us"] == sums).all()
    k = env.array_u64(fds["kcount"])
    assert k[1] == k[4] == len(cost) and k[5] == 12          # one STEAL probe per worker, then retire


def test_spec_examples():
    """SPEC.md: 8 equal units, 4 workers -> 2 per deque; 100 units, 1 worker -> all on it."""
    r, _, _ = _run("fixed", np.full(8, 10), np.arange(8) % 4, 4)
    assert np.bincount(r["executed_by"], minlength=4).tolist() == [2, 2, 2, 2] and r["makespan_us"] == 20
    r, _, _ = _run("greedy", np.full(100, 3), np.zeros(100), 1)
    assert (r["executed_by"] == 0).all() and r["makespan_us"] == 300


def test_victim_is_largest_then_lowest_id():
    """Worker 0 idle; deques [0, 4, 4] -> it steals worker 1's tail unit first."""
    cost = np.full(8, 10)
    home = np.array([1, 1, 1, 1, 2, 2, 2, 2])
    r, _, _ = _run("greedy", cost, home, 3)
    assert r["stolen"][3] == 1 and r["executed_by"][3] == 0      # unit 3 = worker 1's tail


@pytest.mark.parametrize("kind", ["moderate", "heavy"])
def test_greedy_invariants(kind):
    """Every unit exactly once; busy = work; with free stealing Greedy never loses to FixedWork."""
    cost, home = sched.workload(kind, 16)
    g, env, fds = _run("greedy", cost, home, 16)
    f, _, _ = _run("fixed", cost, home, 16)
    assert int(g["busy_us"].sum()) == int(cost.sum())
    assert g["makespan_us"] <= f["makespan_us"]
    assert (g["executed_by"][g["stolen"] == 0] == home[g["stolen"] == 0]).all()
    k = env.array_u64(fds["kcount"])
    assert k[1] == k[4] == len(cost)


def test_latency_budget_caps_stolen_work():
    """LatencyBudget: a worker stops stealing once its stolen work reaches the budget (it may
    overshoot by the last unit it took), and stolen_us records exactly that work."""
    cost, home = sched.workload("heavy", 16)
    budget = 40
    r, env, fds = _run("latency_budget", cost, home, 16, budget=budget)
    stolen_work = np.bincount(r["executed_by"][r["stolen"] == 1], weights=cost[r["stolen"] == 1], minlength=16)
    assert (env.array_u64(fds["stolen_us"]) == stolen_work).all()
    last = np.zeros(16)
    for u in np.nonzero(r["stolen"])[0]:
        last[r["executed_by"][u]] = max(last[r["executed_by"][u]], cost[u])
    assert (stolen_work <= budget + last).all()


def test_max_steals_hand_example():
    """MaxSteals with cap 1 on the victim example, timeline worked by hand (equal 10-us
    units, free steals, lowest id first at equal times): w0 steals unit 3 at t=0, is refused at 10;
    w1 runs 0,1,2 then steals unit 7 from w2 at t=30 (w1 moves before w2 at t=30) and is refused at
    40; w2 runs 4,5,6, is granted at 30 but finds nothing.  Greedy instead has w0 steal unit 7 at 10."""
    cost = np.full(8, 10)
    home = np.array([1, 1, 1, 1, 2, 2, 2, 2])
    r, env, fds = _run("max_steals", cost, home, 3, max_steals=1)
    assert r["executed_by"].tolist() == [1, 1, 1, 0, 2, 2, 2, 1]
    assert r["stolen"].tolist() == [0, 0, 0, 1, 0, 0, 0, 1]
    assert r["steals"].tolist() == [1, 1, 0] and r["makespan_us"] == 40
    assert env.array_u64(fds["steals"]).tolist() == [1, 1, 1]       # granted decisions
    g, _, _ = _run("greedy", cost, home, 3)
    assert g["executed_by"][7] == 0


@pytest.mark.parametrize("kind", ["moderate", "heavy"])
def test_max_steals_limits(kind):
    """Cap 0 is FixedWork; a cap >= the unit count is Greedy; any cap bounds each worker's steals."""
    cost, home = sched.workload(kind, 16)
    f, _, _ = _run("fixed", cost, home, 16, steal_cost=2)
    g, _, _ = _run("greedy", cost, home, 16, steal_cost=2)
    m0, _, _ = _run("max_steals", cost, home, 16, steal_cost=2, max_steals=0)
    mi, _, _ = _run("max_steals", cost, home, 16, steal_cost=2, max_steals=len(cost))
    for a, b in ((m0, f), (mi, g)):
        assert (a["executed_by"] == b["executed_by"]).all() and a["makespan_us"] == b["makespan_us"]
    for cap in (1, 2, 3):
        r, env, fds = _run("max_steals", cost, home, 16, steal_cost=2, max_steals=cap)
        granted = env.array_u64(fds["steals"])
        assert (r["steals"] <= cap).all() and (granted <= cap).all()
        assert ((granted - r["steals"]) <= 1).all()                  # at most one granted attempt finds nothing
