mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for M in "0 0" "3 4"; do set -- $M
GX_JIT_STAGE_MODE=$1 GX_JIT_STAGES=$2 timeout 900 python -m pytest tests -m gpu -x -q -k "jit or overlapped or perthread" > gpurun_out/sweep_tests_$1.log 2>&1; echo mode $1 tests rc=$?; tail -3 gpurun_out/sweep_tests_$1.log
done
for V in "2 4" "3 3" "3 4" "3 6"; do set -- $V
  echo "== mode $1 stages $2"
  GX_JIT_UNROLL=1 GX_JIT_STAGE_MODE=$1 GX_JIT_STAGES=$2 timeout 300 python tools/time_variants.py 28 exit,ctx_sum,p2,p1
  GX_JIT_UNROLL=1 GX_JIT_STAGE_MODE=$1 GX_JIT_STAGES=$2 timeout 300 python tools/time_configs.py C2:30 C4:28 C3:28 C5:26 C1:20 C1:26
done 2>&1 | tee gpurun_out/sweep7.log
