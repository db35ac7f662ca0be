# JIT staging sweep: parity subset then timing per (GX_JIT_STAGE_MODE, GX_JIT_STAGES) (tuning helper; not the bench)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for M in ${MODES:-2}; do
  GX_JIT_STAGE_MODE=$M timeout 900 python -m pytest tests -m gpu -x -q -k "jit" > gpurun_out/sweep_tests_$M.log 2>&1; echo mode $M tests rc=$?; tail -3 gpurun_out/sweep_tests_$M.log
done
for M in ${MODES:-2}; do for S in ${STAGES:-0 2 3 4 6}; do
  echo "== mode $M stages $S"
  GX_JIT_STAGE_MODE=$M GX_JIT_STAGES=$S timeout 300 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C3:28 C5:26 C1:20}
done; done 2>&1 | tee gpurun_out/sweep.log
