mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "prefetch or daemon" > gpurun_out/f2_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/f2_tests.log
timeout 900 python -c "
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench; bench.f2_lines()" 2>&1 | grep '"f2"'
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/C3_jit_full -f python tools/time_configs.py C3:26 > gpurun_out/ncu_C3.log 2>&1; echo ncu rc=$?
