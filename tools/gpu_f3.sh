mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "sched or instrument" > gpurun_out/f3_tests.log 2>&1; echo tests rc=$?; tail -30 gpurun_out/f3_tests.log
timeout 600 python -c "
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench; bench.f3_lines()" 2>&1 | tail -5
