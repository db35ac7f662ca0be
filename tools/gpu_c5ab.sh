# Experiment record (profiles/r2_ptkc.md): the knobs it sets existed only in measurement builds and were removed afterwards.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
  for v in "GX_JIT_NOINLINE=0" "GX_JIT_NOINLINE=1" "GX_JIT_NOINLINE=1 GX_JIT_PTKC=2"; do
    env $v timeout 300 python tools/time_configs.py C5:28 | sed "s/^/$v /"
  done
done
