# Differential fuzz + bounds mode + strict soundness on the GPU.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_bounds.py tests/test_gpu_strict.py -q > gpurun_out/t_fuzz.log 2>&1; echo fuzz rc=$?
tail -40 gpurun_out/t_fuzz.log | grep -v "^E   " | tail -25
grep -o "seed [0-9]*" gpurun_out/t_fuzz.log | sort -u | head
