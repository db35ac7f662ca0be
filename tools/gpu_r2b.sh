# Round-2 features on the GPU: new tests first, then the PTKC / narrow A/B and C1 ingest variants.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_prefetch.py tests/test_gpu_instrument.py tests/test_gpu_aux.py -x -q > gpurun_out/t_new.log 2>&1; echo new tests rc=$?
tail -15 gpurun_out/t_new.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "different_streams or overlapped or c2 or C2 or fuzz" > gpurun_out/t_par.log 2>&1; echo parity rc=$?
tail -5 gpurun_out/t_par.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/t_full.log 2>&1; echo fullsize rc=$?
tail -5 gpurun_out/t_full.log
bash tools/gpu_ab_r2.sh 2>&1 | grep -v "^build"
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py -x -q > gpurun_out/t_san.log 2>&1; echo sanitizer rc=$?
tail -40 gpurun_out/t_san.log
