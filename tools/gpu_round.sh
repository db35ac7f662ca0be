# Round measurement on one B200: smoke, full GPU suite, bench line, extra configs, ncu launch list
# and one full ncu capture of the bench kernel (outputs under gpurun_out/, summarised into profiles/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 900 python bench.py --extra --no-cpu --no-e2e --no-c1 > gpurun_out/extra.json 2> gpurun_out/extra.err; echo extra rc=$?
grep '^{' gpurun_out/extra.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-c1 > gpurun_out/launches.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/bench_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c1 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
