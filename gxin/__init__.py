"""gxin -- the seeded INPUT generators shared by the CUDA path and the CPU oracle.

This module is the only code both sides may use (task rule ③): it produces
*inputs* -- eBPF program bytes (`asm`, `programs`) and synthetic event batches
(`gen`) -- and holds none of the method's arithmetic (no interpretation, no map
semantics, no verification).  Neither `oracle/` nor `paper_2512_12615_b200/`
is imported from here.
"""
from . import asm, gen, programs  # noqa: F401
