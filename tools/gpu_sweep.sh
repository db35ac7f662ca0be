# JIT tuning sweep on one B200 (a helper, not the bench): for each setting in $SWEEP (space-separated
# "VAR=value,VAR=value" groups, e.g. SWEEP="GX_JIT_STAGES=3 GX_JIT_STAGES=4,GX_JIT_RING_RELEASE=mbar")
# time $CONFIGS with tools/time_configs.py.  Knobs: GX_JIT_STAGES, GX_JIT_STAGE_MODE (0-3),
# GX_JIT_RING_RELEASE (atom|mbar), GX_JIT_INGEST (ring|reg), GX_JIT_UNROLL, GX_JIT_BLOCK, GX_JIT_MINB,
# GX_JIT_IFCONV, GX_JIT_PTCACHE, GX_JIT_HASH_L1PROBE, GX_JIT_WAIT_HINT.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for S in ${SWEEP:-GX_JIT_STAGES=3}; do
  echo "== $S"
  env $(echo "$S" | tr ',' ' ') timeout 300 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C3:28 C5:26 C1:20}
done 2>&1 | tee gpurun_out/sweep.log
