timeout 300 python tools/c3_probe.py 28 p3,fetch_array,lookup_only 2>&1 | grep "^{"
C3_TRACES=uniform timeout 300 python tools/c3_probe.py 28 p3,array_only 2>&1 | grep "^{"
for st in 3 4; do echo "stages $st"; GX_JIT_STAGES=$st timeout 300 python tools/c3_probe.py 28 p3 2>&1 | grep "^{"; done
echo "reg ingest"; GX_JIT_INGEST=reg timeout 300 python tools/c3_probe.py 28 p3 2>&1 | grep "^{"
