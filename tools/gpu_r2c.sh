# Round-2 checkpoint: A/B of the block-entry narrowing, config timings, bench line, full GPU suite.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
for rep in 1 2; do
  for k in 1 0; do
    GX_JIT_NARROW=$k timeout 300 python tools/time_configs.py C4:28 C3:28 C5:28 | sed "s/^/narrow=$k /"
  done
done
timeout 300 python tools/time_configs.py C2:30 C1:26 | sed "s/^/default /"
timeout 900 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo bench rc=$?
cat gpurun_out/bench_r2c.json
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2c.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gputests_r2c.log
