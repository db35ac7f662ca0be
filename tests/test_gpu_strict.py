"""Strict-mode soundness on the GPU (SURVEY.md §8c c.7 "Strict-mode soundness"):
a program the verifier accepts with simt_strict = 1 (branch conditions, loop
bounds, shared-map update keys and atomic targets all warp-uniform), run on batches that honour the
UNIFORM contract of §8b (every UNIFORM field equal across a warp record), never splits a warp:
the interpreter's min-PC path reports divergent_steps == 0.  The same batches on the JIT with
GX_JIT_UNIFORM_CHECK=1 check the relaxed-mode divergence analysis: no branch it marked GXF_UNIFORM
ever splits.  Results stay bit-exact with the oracle.

Programs: hand-written uniform loops and the first 60 generated fuzz programs (gxin/fuzzprog.py)
that strict mode admits.  (The config policies are relaxed-mode programs: P1 / P2 / P3 / P4 update
maps at lane-varying keys, which strict mode rejects as NON_UNIFORM_ATOMIC / UNIFORM_MAP_KEY.)"""
import os

import numpy as np
import pytest

import paper_2512_12615_b200 as gx
from gxin import asm, configs, fuzzprog as fp
from oracle.oracle import Oracle
import fuzz_util as fu

pytestmark = pytest.mark.gpu

UNIFORM_LOOPS = [
    # loop bound from a UNIFORM ctx field (size), counter from a constant
    """ldxw r6, [r1+28]
       and64 r6, 15
       mov64 r7, 0
       mov64 r0, 0
       jeq r6, 0, done
    loop:
       add64 r7, r6
       add64 r0, 3
       sub64 r6, 1
       jne r6, 0, loop
    done:
       add64 r0, r7
       exit""",
    # nested: a uniform branch on block_id inside a counted loop
    """ldxw r6, [r1+20]
       mov64 r8, 4
       mov64 r0, 0
    outer:
       mov64 r2, r6
       and64 r2, 1
       jeq r2, 0, even
       add64 r0, 7
       ja next
    even:
       add64 r0, 1
    next:
       rsh64 r6, 1
       sub64 r8, 1
       jsgt r8, 0, outer
       exit""",
]


def _strict_ok(text, fds, specs):
    v, _, _ = gx.gx_verify_offline(asm.assemble(text, fds), {fds[k]: s for k, s in specs.items()}, strict=True)
    return v == 0


def _run(engine, texts, ev, seed, check=False):
    import torch
    from gpu_util import make_runtime
    if check:
        os.environ["GX_JIT_UNIFORM_CHECK"] = "1"
    try:
        rt = make_runtime(engine)
        fds, prog = fu.setup(rt, texts, seed)
        ret = torch.zeros(len(ev), dtype=torch.int64, device="cuda")
        rt.run(torch.from_numpy(ev.view(np.uint8).reshape(-1, 32)).cuda(), prog, ret=ret)
        torch.cuda.synchronize()
        out = fu.outputs(rt, fds, keep_stats=True)
        st = out.pop("_stats")
        rt.close()
    finally:
        os.environ.pop("GX_JIT_UNIFORM_CHECK", None)
    return ret.cpu().numpy().view(np.uint64), out, st["divergent_steps"]


def _oracle(texts, ev, seed):
    env = Oracle()
    fds, prog = fu.setup(env, texts, seed)
    return env.run(ev, prog), fu.outputs(env, fds)


def _strict_fuzz_programs(limit):
    fds = {name: i + 3 for i, name in enumerate(fp.MAPS)}
    out = []
    for seed in range(20000):
        t = fp.program(500000 + seed)
        if _strict_ok(t, fds, fp.MAPS):
            out.append(t)
            if len(out) >= limit:
                break
    return out


@pytest.mark.parametrize("engine", ["interp", "jit"])
def test_strict_programs_never_split(gpu, engine):
    fds = {name: i + 3 for i, name in enumerate(fp.MAPS)}
    texts = [t for t in UNIFORM_LOOPS if _strict_ok(t, fds, fp.MAPS)]
    assert len(texts) == len(UNIFORM_LOOPS)
    texts += _strict_fuzz_programs(60)
    assert len(texts) >= 20, len(texts)
    for k, t in enumerate(texts):
        ev = fp.events(700 + k, 4096 + 7, contract=True)
        r0o, oo = _oracle([t], ev, 700 + k)
        r0g, og, split = _run("interp" if engine == "interp" else "jit", [t], ev, 700 + k, check=engine == "jit")
        assert split == 0, (engine, "warp split on a strict-accepted program", t)
        assert (r0o == r0g).all(), (engine, "R0", t)
        assert oo == og, (engine, "maps", t)
