mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for st in 3 4 5 6; do
  GX_JIT_STAGES=$st timeout 300 python tools/time_configs.py C2:30 C3:28 C5:28 C1:26 | sed "s/^/stages=$st /" | cut -c1-100
done
done
