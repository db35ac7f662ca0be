"""Auxiliary subsystems: GX_LOG_LEVEL logging from the runtime (errors, JIT compiles,
launches) -- checked in a subprocess so the level is read fresh."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2512_12615_b200 as gx
from gxin import configs
rt = gx.Runtime(0)
s = configs.setup(rt, "C1")
ev = torch.from_numpy(configs.events("C1", 1, 4096).view(np.uint8).reshape(-1, 32)).cuda()
rt.run(ev, s.prog_arg)
torch.cuda.synchronize()
try:
    rt.update_map(s.fds[(0, "counts")], b"\0" * 4, b"\0" * 8, 7)   # bad flags -> -EINVAL
    gx.gx_attach(rt.rt, 99, 0, 0)                                     # no such program
except Exception:
    pass
print("done")
""" % ROOT


@pytest.mark.parametrize("level", [0, 1, 3])
def test_log_level(gpu, level):
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, GX_LOG_LEVEL=str(level)))
    assert r.returncode == 0 and "done" in r.stdout, r.stderr[-2000:]
    err = r.stderr
    assert ("[gx:2] JIT variant" in err) == (level >= 2)
    assert ("[gx:3] batch 0: 4096 events" in err) == (level >= 3)
    if level == 0:
        assert "[gx:" not in err


def test_jit_failure_falls_back_to_the_interpreter(gpu, monkeypatch):
    """A launch configuration the JIT cannot compile runs on the interpreter (same GPU, same
    semantics): GX_JIT_INJECT_FAILURE makes every compile fail; C3 still matches the oracle and the
    interpreter's warp steps show it ran."""
    import numpy as np
    import torch
    from gxin import configs
    from gpu_util import make_runtime, oracle_run, outputs
    monkeypatch.setenv("GX_JIT_INJECT_FAILURE", "1")
    n = 4096 + 17
    ev = configs.events("C3", configs.SEEDS["C3"], n)
    env, so, r0o = oracle_run("C3", ev, threshold=2)
    rt = make_runtime("jit")
    s = configs.setup(rt, "C3", threshold=2)
    ret = torch.zeros(n, dtype=torch.int64, device="cuda")
    rt.run(torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda(), s.prog_arg, ret=ret)
    torch.cuda.synchronize()
    st = rt.stats()
    assert (ret.cpu().numpy().view(np.uint64) == r0o).all()
    assert outputs(rt, s) == outputs(env, so)
    assert st["warp_steps"] > 0
