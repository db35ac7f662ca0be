mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
GX_JIT_CLAIM=2 GX_JIT_INGEST=ring timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tools/time_configs.py C2:22 2>&1 | head -40; GX_JIT_CLAIM=2 timeout 300 python tools/time_configs.py C2:24 C2:26 C2:28 2>&1 | tail -5
