# Round measurement: smoke, full GPU suite, bench line, extra lines, launch list, ncu of the bench kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_final.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gputests_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
cat gpurun_out/bench_final.json
timeout 1200 python bench.py --extra --no-cpu --no-e2e --no-c1 --no-configs --steps 3 > gpurun_out/extra_final.json 2> gpurun_out/extra_final.err; echo extra rc=$?
grep '^{' gpurun_out/extra_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-c1 --no-configs > gpurun_out/launches.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/bench_final_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c1 --no-configs > gpurun_out/ncu_final.log 2>&1; echo ncu rc=$?
