mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for P in 0 1; do echo "== ptcache $P"; GX_JIT_PTCACHE=$P timeout 600 python tools/time_variants.py 30; done 2>&1 | tee gpurun_out/variants.log
GX_JIT_PTCACHE=0 timeout 900 ncu --set full --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/c2_jit_full -f python tools/time_configs.py C2:30 > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_c2.log
