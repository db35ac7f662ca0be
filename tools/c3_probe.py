"""C3 bottleneck probe (tuning helper, not the bench): P3 variants on (a) the C3 trace and (b) the same
trace with its pages remapped uniformly at random (no hot pages).  python tools/c3_probe.py [lg_n]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_12615_b200 as gx  # noqa: E402
from gxin import asm, configs, gen_gpu, programs  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from time_c3_variants import VARIANTS  # noqa: E402  (module body runs with argv -> guarded below)

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
only = [x for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["p3", "fetch", "red", "fetch_array", "array_only", "lookup_only"]) if x in VARIANTS]
ev = gen_gpu.generate_device("C3", configs.SEEDS["C3"], n)
evu = ev.clone()
a64 = evu.view(torch.int64).view(-1, 4)
g = torch.Generator(device="cuda").manual_seed(1)
pages = torch.randint(0, 1 << 20, (n,), device="cuda", generator=g, dtype=torch.int64)
a64[:, 0] = pages << 12
TRACES = os.environ.get("C3_TRACES", "c3").split(",")
for trace, E in [(t, {"c3": ev, "uniform": evu}[t]) for t in TRACES]:
    for name in only:
        text = VARIANTS[name]
        rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT)
        fds = {k: rt.create_map(s.type, s.key_size, s.value_size, s.max_entries) for k, s in programs.P3_MAPS.items()}
        fds["cnt"] = rt.create_map(programs.ARRAY, 4, 8, 1 << 20)
        fds["cnt16"] = rt.create_map(programs.ARRAY, 4, 16, 1 << 20)
        fds["cnt2"] = rt.create_map(programs.ARRAY, 4, 8, 1 << 21)
        fds["cnt216"] = rt.create_map(programs.ARRAY, 4, 16, 1 << 21)
        fd = rt.load_prog(asm.assemble(text, fds))
        for _ in range(3):
            rt.run(E, fd)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            rt.run(E, fd)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        print(json.dumps({"trace": trace, "n": n, "prog": name, "ms": round(ms, 4), "hash_full": rt.stats()["hash_full"]}), flush=True)
        rt.close()

if os.environ.get("C3_NOHOT"):
    # the same trace with the K hottest pages' events skipping the map (their FETCH-ADDs removed):
    # how much of C3 is the same-address serialisation on its hot pages
    pg = (ev.view(torch.int64).view(-1, 4)[:, 0] >> 12)
    cnt = torch.bincount(pg, minlength=1 << 20)
    for K in [int(x) for x in os.environ["C3_NOHOT"].split(",")]:
        top = torch.topk(cnt, K).indices.tolist() if K else []
        skip = "".join(f"    jeq r6, {p}, out\n" for p in top)
        text = programs.P3.replace("    rsh64 r6, 12              ; page\n", "    rsh64 r6, 12              ; page\n" + skip)
        rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT)
        fds = {k: rt.create_map(s.type, s.key_size, s.value_size, s.max_entries) for k, s in programs.P3_MAPS.items()}
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
        share = float(cnt[top].sum()) / n if K else 0.0
        print(json.dumps({"trace": "c3", "prog": f"p3 minus top {K} pages", "events_share": round(share, 4),
                          "ms": round(a.elapsed_time(b) / 5, 4)}), flush=True)
        rt.close()
