# Round-2 A/B: per-thread key cache (GX_JIT_PTKC) on C2/C4/C5, C1 single-launch ingest variants.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
for rep in 1 2; do
  for k in 1 0; do
    GX_JIT_PTKC=$k timeout 300 python tools/time_configs.py C2:30 C5:28 C4:28 | sed "s/^/ptkc=$k /"
  done
done
for v in "" "GX_JIT_INGEST=ring GX_JIT_STAGES=2" "GX_JIT_INGEST=ring GX_JIT_STAGES=3" "GX_JIT_INGEST=ring GX_JIT_STAGES=4" "GX_JIT_EPT=4" "GX_JIT_EPT=16"; do
  env $v timeout 120 python tools/time_c1.py C1
done
