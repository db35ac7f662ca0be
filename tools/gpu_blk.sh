mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for b in 1024 768 512; do
  GX_JIT_BLOCK=$b timeout 300 python tools/time_configs.py C5:28 C4:28 C3:28 | sed "s/^/block=$b /"
done
done
