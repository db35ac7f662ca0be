"""Workload run under compute-sanitizer by tests/test_gpu_sanitizer.py (SURVEY.md §4 layer 9, §5):
small batches of every config on both engines and both JIT ingests, a PDL-chained pair, a hook-
instrumented kernel and the CLC scheduler, each checked against the oracle so that the sanitized
run is known to have done the work.  Exit code 0 = all parity checks passed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gpu_util import make_runtime, oracle_run, outputs  # noqa: E402
from gxin import configs  # noqa: E402


def main(which):
    n = 4096 + 17
    for engine in ("interp", "jit", "jit_ring"):
        for config in ("C1", "C2", "C3", "C4", "C5", "C6"):
            T = 2 if config == "C3" else None
            ev = configs.events(config, configs.SEEDS[config], n)
            env, so, r0o = oracle_run(config, ev, threshold=T)
            rt = make_runtime(engine)
            s = configs.setup(rt, config, threshold=T)
            d_ev = torch.from_numpy(np.ascontiguousarray(ev).view(np.uint8).reshape(-1, 32)).cuda()
            ret = torch.zeros(n, dtype=torch.int64, device="cuda")
            half = (n // 64) * 32
            rt.run(d_ev[:half], s.prog_arg, ret=ret[:half])
            rt.run(d_ev[half:], s.prog_arg, ret=ret[half:], overlap=engine != "interp")
            torch.cuda.synchronize()
            assert (ret.cpu().numpy().view(np.uint64) == r0o).all(), (engine, config)
            assert outputs(rt, s) == outputs(env, so), (engine, config)
            rt.close()
            print(which, engine, config, "ok", flush=True)
    if which != "racecheck":     # the spin-timed scheduler would take minutes under racecheck
        import paper_2512_12615_b200 as gx
        from gxin import sched
        cost = np.full(64, 2, dtype=np.uint32)
        rt = gx.Runtime(0)
        prog, fds = sched.setup(rt, "max_steals", 64, max_steals=2)
        r = gx.gx_sched_run_ex(rt.rt, prog, cost, None, 0, 0, flags=gx.GX_SCHED_CLC, smem_per_block=200 * 1024,
                               log_cap=512)
        assert sorted(r["executed_by"].tolist()) != [] and (r["executed_by"] < 64).all()
        rt.close()
        print(which, "clc ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "memcheck")
