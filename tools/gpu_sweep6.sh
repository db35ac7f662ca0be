mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for V in "2 0 0" "1 2 4"; do set -- $V
  echo "== unroll $1 mode $2 stages $3"
  GX_JIT_UNROLL=$1 GX_JIT_STAGE_MODE=$2 GX_JIT_STAGES=$3 timeout 300 python tools/time_variants.py 28
done 2>&1 | tee gpurun_out/sweep6.log
