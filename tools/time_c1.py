"""C1 (2^20-event counter batches) single-launch and CUDA-graph steady-state timing with rotation
over 8 batches (256 MiB > L2) -- tuning helper."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_12615_b200 as gx  # noqa: E402
from gxin import configs, gen_gpu  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "C1"
n, nb = 1 << 20, 8
rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT)
s = configs.setup(rt, config)
bufs = [gen_gpu.generate_device(config, configs.SEEDS[config], n, i0=k * n, n_total=nb * n) for k in range(nb)]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for k in range(24):
        rt.run(bufs[k % nb], s.prog_arg, stream=st)
    st.synchronize()
    ts = []
    for k in range(40):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        rt.run(bufs[k % nb], s.prog_arg, stream=st)
        b.record(st)
        ts.append((a, b))
    st.synchronize()
    single = float(np.median([a.elapsed_time(b) for a, b in ts])) * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for k in range(100):
            rt.run(bufs[k % nb], s.prog_arg, stream=st)
    g.replay()
    st.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(5):
        g.replay()
    b.record(st)
    st.synchronize()
    steady = a.elapsed_time(b) / 500 * 1e3
env = {k: v for k, v in os.environ.items() if k.startswith("GX_")}
print(json.dumps({"config": config, "env": env, "single_us": round(single, 2), "steady_us": round(steady, 2),
                  "steady_frac": round(5.127 / steady, 3), "grid": gx.gx_exec_info(rt.rt)["grid"]}), flush=True)
