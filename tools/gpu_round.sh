set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 600 python bench.py --extra --no-cpu --no-e2e > gpurun_out/extra.json 2> gpurun_out/extra.err; echo extra rc=$?
tail -20 gpurun_out/extra.err
