mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomic_bench tools/atomic_bench.cu && /tmp/atomic_bench > gpurun_out/atomics_b200.json; cat gpurun_out/atomics_b200.json
timeout 1500 python -m pytest tests -m gpu -x -q -k "prefetch or daemon or merge or overlapped or full_size" > gpurun_out/f2_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/f2_tests.log
timeout 900 python bench.py --no-e2e --no-cpu --extra > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/f2_bench.json')); print(d['value'], d['roofline']['frac'], json.dumps(d['c1']))"
grep '"f2"' gpurun_out/f2_bench.err
