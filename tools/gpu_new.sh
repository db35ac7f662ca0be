# New-feature GPU check: build, f3 (sched log replay, CLC) + f2 L2 + f4 tests, then the extra bench lines.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_prefetch.py tests/test_gpu_instrument.py -x -q > gpurun_out/new_tests.log 2>&1; echo tests rc=$?
tail -30 gpurun_out/new_tests.log
timeout 900 python bench.py --extra --no-cpu --no-e2e --no-c1 --no-configs --steps 3 --warmup 3 > gpurun_out/extra_new.json 2> gpurun_out/extra_new.err; echo extra rc=$?
grep '^{' gpurun_out/extra_new.err | grep -v '"config"'
