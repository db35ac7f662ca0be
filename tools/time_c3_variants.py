"""What bounds C3: the same 2^28 C3 events under P3 variants (tuning helper; maps persist across the
warm-up, so timed runs are lookups + FETCH-ADDs on a populated table, as in tools/time_configs.py).
    python tools/time_c3_variants.py [lg_n] [variant,...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_12615_b200 as gx  # noqa: E402
from gxin import asm, configs, gen_gpu, programs  # noqa: E402

P3 = programs.P3
HEAD = P3.split("have:")[0] + "have:\n"
VARIANTS = {
    "p3": P3,
    "lookup_only": HEAD + "    mov64 r0, 0\n    exit\nout:\n    mov64 r0, 0\n    exit\n",
    "red": HEAD + "    mov64 r1, 1\n    atomic_add64 [r0+0], r1\nout:\n    mov64 r0, 0\n    exit\n",
    "fetch": HEAD + "    mov64 r1, 1\n    atomic_fetch_add64 [r0+0], r1\n    mov64 r0, r1\n    exit\nout:\n    mov64 r0, 0\n    exit\n",
    "page_only": "ldxdw r0, [r1+0]\nrsh64 r0, 12\nexit",
    # the same probe, the FETCH-ADD on a per-page counter in a separate ARRAY (another cache line than
    # the key): what the key/value line sharing costs
    "fetch_array": HEAD + """    mov64 r2, r6
    and64 r2, 1048575
    stxw [r10-12], r2
    lddw r1, map:cnt
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, out
    mov64 r1, 1
    atomic_fetch_add64 [r0+0], r1
    mov64 r0, r1
    exit
out:
    mov64 r0, 0
    exit
""",
    # the FETCH-ADD target laid out like the hash slots' value words, without keys in the lines:
    # 16-B stride at offset 8 (arr16), slot index = a multiplicative hash of the page (hidx, hidx16)
    "fetch_arr16": HEAD + """    mov64 r2, r6
    and64 r2, 1048575
    stxw [r10-12], r2
    lddw r1, map:cnt16
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, out
    mov64 r1, 1
    atomic_fetch_add64 [r0+8], r1
    mov64 r0, r1
    exit
out:
    mov64 r0, 0
    exit
""",
    "fetch_hidx": HEAD + """    lddw r2, 0x9E3779B97F4A7C15
    mul64 r2, r6
    rsh64 r2, 43
    stxw [r10-12], r2
    lddw r1, map:cnt2
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, out
    mov64 r1, 1
    atomic_fetch_add64 [r0+0], r1
    mov64 r0, r1
    exit
out:
    mov64 r0, 0
    exit
""",
    "fetch_hidx16": HEAD + """    lddw r2, 0x9E3779B97F4A7C15
    mul64 r2, r6
    rsh64 r2, 43
    stxw [r10-12], r2
    lddw r1, map:cnt216
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, out
    mov64 r1, 1
    atomic_fetch_add64 [r0+8], r1
    mov64 r0, r1
    exit
out:
    mov64 r0, 0
    exit
""",
    "array_only": """    ldxdw r6, [r1+0]
    rsh64 r6, 12
    and64 r6, 1048575
    stxw [r10-12], r6
    lddw r1, map:cnt
    mov64 r2, r10
    add64 r2, -12
    call 1
    jeq r0, 0, out
    mov64 r1, 1
    atomic_fetch_add64 [r0+0], r1
    mov64 r0, r1
out:
    exit
""",
}
if __name__ == "__main__":
    n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 28)
    ONLY = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    ev = gen_gpu.generate_device("C3", configs.SEEDS["C3"], n)
    for name, text in VARIANTS.items():
        if ONLY and name not in ONLY:
            continue
        rt = gx.Runtime(0, engine=gx.GX_ENGINE_JIT)
        fds = {k: rt.create_map(s.type, s.key_size, s.value_size, s.max_entries) for k, s in programs.P3_MAPS.items()}
        fds["cnt"] = rt.create_map(programs.ARRAY, 4, 8, 1 << 20)
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
        print(json.dumps({"events": "C3", "n": n, "prog": name, "ms": round(ms, 4),
                          "ev_per_s": round(n / (ms / 1e3), 1)}), flush=True)
        rt.close()
