mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for C in ${NCU_CONFIGS:-C2:30 C3:26}; do
  n=${C%%:*}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/${n}_jit_full -f python tools/time_configs.py $C > gpurun_out/ncu_$n.log 2>&1; echo ncu $C rc=$?
done
