# Shared-memory carve-out check (helper): which carve-out the driver picks for the ring kernel (ncu
# launch statistics), then the ring depth x carve-out sweep of tools/gpu_sweep2.sh.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for CO in "" 0; do
  GX_JIT_CARVEOUT=$CO timeout 300 ncu --section LaunchStats --section Occupancy -k regex:gx_jit -c 1 \
    python tools/time_configs.py C2:24 2>&1 | grep -i "shared memory\|L1\|Driver\|Block Limit" | sed "s/^/[carve=$CO] /"
done | tee gpurun_out/carve.log
bash tools/gpu_sweep2.sh
