"""Dump the JIT source + cubin of one config program offline: python tools/jit_dump.py P2 (GX_JIT_DUMP_CUBIN=path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, os
import paper_2512_12615_b200 as gx
from gxin import programs
name=sys.argv[1]
specs = programs.maps_of(name)
fds = {k: i for i, k in enumerate(specs)}
maps = {fds[k]: (s.type, s.key_size, s.value_size, s.max_entries) for k, s in specs.items()}
rc, src, log = gx.gx_jit_offline(programs.build(name, fds), maps)
open(f"/tmp/{name}.cu","w").write(src)
print(rc, log[-500:])
