# PT-cache + staging sweep (tuning helper; not the bench)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_bench tools/atomic_bench.cu && /tmp/atomic_bench > gpurun_out/atomics_b200.json; cat gpurun_out/atomics_b200.json
timeout 900 python -m pytest tests -m gpu -x -q -k "jit" > gpurun_out/sweep_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/sweep_tests.log
for V in "1 0 0" "0 0 0" "1 1 2" "1 2 4" "1 1 3"; do set -- $V
  echo "== ptcache $1 mode $2 stages $3"
  GX_JIT_PTCACHE=$1 GX_JIT_STAGE_MODE=$2 GX_JIT_STAGES=$3 timeout 300 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C5:26 C1:20 C1:26}
done 2>&1 | tee gpurun_out/sweep2.log
