mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for V in "2 0 0" "3 0 0" "4 0 0" "6 0 0" "8 0 0" "1 1 3" "1 1 4" "1 2 4" "1 2 6"; do set -- $V
  echo "== unroll $1 mode $2 stages $3"
  GX_JIT_UNROLL=$1 GX_JIT_STAGE_MODE=$2 GX_JIT_STAGES=$3 timeout 300 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C3:28 C5:26 C1:20 C1:26}
done 2>&1 | tee gpurun_out/sweep5.log
