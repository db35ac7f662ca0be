# Ring-geometry sweep (helper): tools/gpu_sweep.sh over $SWEEP, then the exit-only / P2 program variants
# of tools/time_variants.py under each setting of $VSWEEP (what the event stream alone reaches).
bash tools/gpu_sweep.sh
for S in ${VSWEEP:-GX_JIT_STAGES=3}; do
  echo "== variants $S"
  env $(echo "$S" | tr ',' ' ') timeout 300 python tools/time_variants.py 30 exit,p2
done 2>&1 | tee gpurun_out/vsweep.log
