for v in 0 1 2; do
  echo "== GX_JIT_ATOM_MIXED=$v"
  GX_JIT_ATOM_MIXED=$v timeout 300 python tools/c3_probe.py 28 p3,fetch_array,array_only 2>&1 | grep "^{"
  GX_JIT_ATOM_MIXED=$v C3_TRACES=uniform timeout 300 python tools/c3_probe.py 28 array_only 2>&1 | grep "^{"
done
GX_JIT_ATOM_MIXED=1 timeout 600 python -m pytest -x -q tests/test_gpu_helpers.py -k "bruteforce and jit" 2>&1 | tail -5
