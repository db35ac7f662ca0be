mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "ingest_variants or overlapped or full_size or config_parity or ragged or daemon" > gpurun_out/rel_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/rel_tests.log
for R in mbar atom mbar atom; do echo "== release $R"; GX_JIT_RING_RELEASE=$R timeout 300 python tools/time_configs.py C2:30 C5:26 C3:28 C6:28; done
