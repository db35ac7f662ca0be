# Experiment record (profiles/r2_ptkc.md): the knobs it sets existed only in measurement builds and were removed afterwards.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
timeout 120 python tools/time_c1.py C1
GX_JIT_FLUSH_EXPERIMENT=1 timeout 120 python tools/time_c1.py C1
GX_JIT_FLUSH_EXPERIMENT=2 timeout 120 python tools/time_c1.py C1
done
