# GPU test pass: build, selected pytest files (args), timings. Usage: bash tools/gpu_tests.sh <pytest args>
mkdir -p gpurun_out
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${GX_TEST_TIMEOUT:-2400} python -m pytest -x -q -rA --durations=15 "$@" > gpurun_out/tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|Error|error" gpurun_out/tests.log | tail -5
