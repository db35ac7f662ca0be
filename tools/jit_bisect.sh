#!/bin/bash
# JIT correctness bisection at scale (writes gpurun_out/bisect_*.log)
mkdir -p gpurun_out
i=0
for v in "X=1" "GX_JIT_NOCOOP=1" "GX_JIT_NOWARPAGG=1" "GX_JIT_NOCOOP=1 GX_JIT_NOWARPAGG=1" "GX_JIT_BLOCK=256" "GX_JIT_UNROLL=1"; do
  env $v timeout 150 python tools/debug_cfg.py C3 22 1 > gpurun_out/bisect_$i.log 2>&1
  echo "[$v] rc=$?" >> gpurun_out/bisect_$i.log
  i=$((i+1))
done
