mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python tools/time_configs.py C2:30 C4:28 C3:28 C5:26 C1:26 --engine interp
GX_FUZZ_CASES=2000 timeout 1500 python -m pytest tests/test_gpu_fuzz.py::test_fuzz_interp tests/test_gpu_parity.py -q -k "interp" > gpurun_out/t_interp.log 2>&1; echo interp tests rc=$?; tail -3 gpurun_out/t_interp.log
