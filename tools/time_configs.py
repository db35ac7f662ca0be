"""Quick single-GPU timing of configs (JIT by default) -- a tuning helper, not the bench.
    python tools/time_configs.py C2:28 C1:26 C4:26 [--engine interp]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_12615_b200 as gx  # noqa: E402
from gxin import configs, gen_gpu  # noqa: E402

eng = gx.GX_ENGINE_INTERP if "--engine" in sys.argv and sys.argv[sys.argv.index("--engine") + 1] == "interp" else gx.GX_ENGINE_JIT
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
for spec in [a for a in sys.argv[1:] if ":" in a]:
    config, lg = spec.split(":")
    n = 1 << int(lg)
    rt = gx.Runtime(0, engine=eng)
    s = configs.setup(rt, config)
    ev = gen_gpu.generate_device(config, configs.SEEDS[config], n)
    for _ in range(3):
        rt.run(ev, s.prog_arg)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        rt.run(ev, s.prog_arg)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    st = rt.stats()
    print(json.dumps({"config": config, "n": n, "unroll": os.environ.get("GX_JIT_UNROLL", "2"), "ms": round(ms, 4),
                      "ev_per_s": n / ms * 1e3, "hbm_frac": round(32 * n / (ms / 1e3) / 1e9 / peak, 4),
                      "grid": gx.gx_exec_info(rt.rt)["grid"], "block": gx.gx_exec_info(rt.rt)["block"],
                      "run_ok": st["events_run"] == 8 * n, "hash_full": st["hash_full"],
                      "rb_drops": st["ringbuf_drops"]}), flush=True)
    del ev
    rt.close()
