"""HASH insert storm timing (exact capacity, I-22): N events over K keys into a map of
max_entries M, per engine; prints ms, refusals, entries.  python tools/storm_probe.py"""
import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
from gxin import asm, gen
from gpu_util import make_runtime
import test_gpu_helpers as t
for engine in ("interp", "jit"):
    for K, M in ((1000, 1000), (1000, 4096), (60000, 65536)):
        for rep in range(2):
            n = 64000
            rng = np.random.default_rng(5 + rep)
            keys = (rng.permutation(n) % K + 1).astype(np.uint64)
            ev3 = gen.records(n, addr=keys, ts=7)
            rt = make_runtime(engine)
            fd = rt.create_map(1, 8, 8, M)
            p = rt.load_prog(asm.assemble(t.FILL_HASH, {"h": fd}))
            ret3 = torch.zeros(n, dtype=torch.int64, device="cuda")
            d = torch.from_numpy(ev3.view(np.uint8).reshape(-1, 32)).cuda()
            rt.run(d[:32], p)  # compile
            rt2 = make_runtime(engine)
            torch.cuda.synchronize()
            fd = rt.create_map(1, 8, 8, M)
            p = rt.load_prog(asm.assemble(t.FILL_HASH, {"h": fd}))
            rt.run(d[:32], p)
            torch.cuda.synchronize()
            fd2 = rt.create_map(1, 8, 8, M)
            p2 = rt.load_prog(asm.assemble(t.FILL_HASH, {"h": fd2}))
            rt.run(d[:32], p2)
            torch.cuda.synchronize()
            t0 = time.time()
            rt.run(d[32:], p2, ret=ret3[32:])
            torch.cuda.synchronize(); dt = time.time() - t0
            r = ret3[32:].cpu().numpy()
            print(engine, K, M, rep, "ms", round(dt * 1e3, 2), "refused", int((r != 0).sum()), "entries", len(rt.hash_items(fd2)), flush=True)
            rt.close(); rt2.close()
