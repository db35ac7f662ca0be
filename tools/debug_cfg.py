"""Debug helper: run one config on the GPU (JIT unless --interp) at 2^lg events, R times, then check
hash maps for duplicate keys and compare every map with the oracle (small n)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_12615_b200 as gx  # noqa: E402
from gxin import configs, gen_gpu  # noqa: E402

config, lg = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
eng = gx.GX_ENGINE_INTERP if "--interp" in sys.argv else gx.GX_ENGINE_JIT
n = 1 << lg
rt = gx.Runtime(0, engine=eng)
s = configs.setup(rt, config)
ev = gen_gpu.generate_device(config, configs.SEEDS[config], n)
for _ in range(reps):
    rt.run(ev, s.prog_arg)
torch.cuda.synchronize()
st = rt.stats()
print("stats", st, "exec", gx.gx_exec_info(rt.rt))
for (t, name), fd in sorted(s.fds.items()):
    spec = rt.specs[fd]
    if spec[0] == 1:
        items = gx.gx_read_map(rt.rt, fd, spec)
        keys = [k for k, _ in items]
        print(name, "entries", len(keys), "distinct", len(set(keys)))
if n <= (1 << 22) and reps == 1:
    from gpu_util import oracle_run, outputs
    evh = ev.cpu().numpy().view(np.dtype([("addr", "<u8"), ("ts", "<u8"), ("hook", "<u4"), ("block_id", "<u4"),
                                          ("sm_id", "<u2"), ("warp_id", "u1"), ("lane_id", "u1"), ("size", "<u4")])).reshape(-1)
    env, so, _ = oracle_run(config, evh)
    oo, og = outputs(env, so), outputs(rt, s)
    for k in oo:
        print(k, "MATCH" if oo[k] == og[k] else "DIFF")
