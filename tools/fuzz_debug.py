"""Re-run one differential-fuzz case several times on one engine and print what differs
(debug helper).  python tools/fuzz_debug.py SEED [engine] [reps]"""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import fuzz_util as fu
from gxin import fuzzprog as fp
import test_gpu_fuzz as t

seed = int(sys.argv[1]); engine = sys.argv[2] if len(sys.argv) > 2 else "interp"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
texts, ev = fu.case(seed)
r0o, oo = t._oracle(texts, ev, seed)
print("events", len(ev), "programs", len(texts), "oracle stats", oo["stats"])
for rep in range(reps):
    from gpu_util import make_runtime
    rt = make_runtime(engine, set_env=False)
    r0g, og = t._gpu(texts, ev, seed, rt)
    st = og.pop("_stats")
    rt.close()
    bad = [k for k in oo if oo[k] != og[k]]
    line = f"rep {rep}: differs {bad} gpu stats {og['stats']} herr {st['helper_errors']}"
    for k in bad:
        if k in ("hacc", "hacc4", "hobs"):
            ks, vs = fp.MAPS[k][1], fp.MAPS[k][2]
            def ent(raw):
                return {int.from_bytes(raw[i:i + ks], "little"): raw[i + ks:i + ks + vs] for i in range(0, len(raw), ks + vs)}
            a, b = ent(oo[k]), ent(og[k])
            line += f" | {k}: oracle {len(a)} gpu {len(b)} missing {sorted(set(a) - set(b))[:8]} extra {sorted(set(b) - set(a))[:8]}"
            line += f" valdiff {[x for x in a if x in b and a[x] != b[x]][:8]}"
    print(line, flush=True)
