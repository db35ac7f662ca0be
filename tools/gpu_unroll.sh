mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "GX_JIT_UNROLL=2" "GX_JIT_UNROLL=1" "GX_JIT_UNROLL=4" "GX_JIT_PUNROLL=0" "GX_JIT_STAGES=3" "GX_JIT_HASH_CACHE=1024"; do
  env $v timeout 300 python tools/time_configs.py C3:28 C5:28 | sed "s/^/$v /" | cut -c1-110
done
