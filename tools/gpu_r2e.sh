mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests/test_gpu_instrument.py -x -q > gpurun_out/t_instr.log 2>&1; echo instr rc=$?; tail -3 gpurun_out/t_instr.log
timeout 300 python tools/time_configs.py C4:28 C3:28 C5:28 C2:30
timeout 900 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r2e.json')); print(json.dumps(d['c1']))"
