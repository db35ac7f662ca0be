mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "jit or overlapped or perthread" > gpurun_out/quick_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/quick_tests.log
for V in "0 1 3" "1000000 1 3" "0 0 3" "0 1 4" "0 1 0"; do set -- $V
  echo "== hint $1 ifconv $2 stages $3"
  GX_JIT_WAIT_HINT=$1 GX_JIT_IFCONV=$2 GX_JIT_STAGES=$3 timeout 300 python tools/time_configs.py C2:30 C4:28 C3:28 C5:26 C1:20 C1:26
done 2>&1 | tee gpurun_out/sweep9.log
