mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for C in C4:26 C5:26; do n=${C%%:*}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gx_jit -s 3 -c 1 -o gpurun_out/${n}_jit_full -f python tools/time_configs.py $C > gpurun_out/ncu_$n.log 2>&1; echo ncu $C rc=$?
done
for V in "1024 1" "1024 2" "512 3" "512 4" "256 8"; do set -- $V
  echo "== block $1 minb $2"
  GX_JIT_BLOCK=$1 GX_JIT_MINB=$2 timeout 300 python tools/time_configs.py C3:28 C4:28 C5:26 C2:30
done 2>&1 | tee gpurun_out/sweep8.log
