# build, JIT parity subset, timing of every config (tuning helper; not the bench)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-jit}" > gpurun_out/quick_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/quick_tests.log
timeout 600 python tools/time_configs.py ${CONFIGS:-C2:30 C4:28 C3:28 C5:26 C1:20 C1:26} 2>&1 | tee gpurun_out/quick.log
[ -n "$NCU" ] && timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/quick_ncu -f python tools/time_configs.py $NCU > gpurun_out/quick_ncu.log 2>&1
echo done
