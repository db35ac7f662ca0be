"""Isolate what bounds the C2 kernel: the same 2^30 C2 events under program variants (tuning helper).
    python tools/time_variants.py [lg_n]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_12615_b200 as gx  # noqa: E402
from gxin import asm, configs, gen_gpu, programs  # noqa: E402

P2 = programs.P2
HIST_ONLY = P2.split("lane:")[0] + "lane:\n    mov64 r0, 0\n    exit\n"
PT_ONLY = "    mov64 r6, r1\n" + P2.split("lane:")[1]
VARIANTS = {
    "exit": "mov64 r0, 0\nexit",
    "ctx_sum": "ldxdw r0, [r1+0]\nldxdw r2, [r1+8]\nadd64 r0, r2\nldxw r2, [r1+16]\nadd64 r0, r2\nldxw r2, [r1+28]\nadd64 r0, r2\nexit",
    "hist_only": HIST_ONLY,
    "pt_only": PT_ONLY,
    "p2": P2,
    "p1": programs.P1,
    "p1d": programs.P1D,
}
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 30)
ONLY = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for cfg in ("C2", "C1"):
    ev = gen_gpu.generate_device(cfg, configs.SEEDS[cfg], n)
    for name, text in VARIANTS.items():
        if ONLY and name not in ONLY:
            continue
        rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT)
        specs = dict(programs.P2_MAPS)
        specs.update(programs.P1_MAPS if name == "p1" else programs.P1D_MAPS if name == "p1d" else {})
        fds = {k: rt.create_map(s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
        fd = rt.load_prog(asm.assemble(text, fds))
        for _ in range(3):
            rt.run(ev, fd)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            rt.run(ev, fd)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(json.dumps({"events": cfg, "n": n, "prog": name, "ms": round(ms, 4),
                          "hbm_frac": round(32 * n / (ms / 1e3) / 1e9 / peak, 4)}), flush=True)
        rt.close()
    del ev
