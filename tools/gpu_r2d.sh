# Round-2 profiling + full suite: ncu --set full of the bench kernel (C2) and of C3 / C5 / C4, the
# bench launch list, then the whole GPU suite.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/r2_c2_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c1 --no-configs > gpurun_out/ncu_c2.log 2>&1; echo ncu c2 rc=$?
for C in C3:26 C5:26 C4:26; do
  n=${C%%:*}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/r2_${n}_full -f python tools/time_configs.py $C > gpurun_out/ncu_$n.log 2>&1; echo ncu $C rc=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-c1 --no-configs > gpurun_out/launches.log 2>&1; echo launches rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fuzz.py > gpurun_out/gputests_r2d.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gputests_r2d.log
