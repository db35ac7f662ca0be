mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "jit" > gpurun_out/sweep_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/sweep_tests.log
for P in 0 1; do echo "== ptcache $P"; GX_JIT_PTCACHE=$P timeout 600 python tools/time_variants.py 30; done 2>&1 | tee gpurun_out/variants.log
for V in "0 0 0" "0 1 2" "1 0 0"; do set -- $V
  echo "== ptcache $1 mode $2 stages $3"
  GX_JIT_PTCACHE=$1 GX_JIT_STAGE_MODE=$2 GX_JIT_STAGES=$3 timeout 300 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C3:28 C5:26 C1:20 C1:26}
done 2>&1 | tee gpurun_out/sweep3.log
