mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "perthread or isa or micro" > gpurun_out/sweep_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/sweep_tests.log
for V in "1024 1 2" "672 2 2" "672 2 1" "448 3 1" "512 2 1" "640 2 2" "512 3 1"; do set -- $V
  echo "== block $1 minb $2 unroll $3"
  GX_JIT_BLOCK=$1 GX_JIT_MINB=$2 GX_JIT_UNROLL=$3 timeout 300 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C3:28 C5:26 C1:20 C1:26}
done 2>&1 | tee gpurun_out/sweep4.log
