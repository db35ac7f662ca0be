mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "C3 or C5 or hash or micro" > gpurun_out/c3_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/c3_tests.log
for P in 1 0; do echo "== l1probe $P"; GX_JIT_HASH_L1PROBE=$P timeout 300 python tools/time_configs.py C3:28 C5:26 C3:26; done
