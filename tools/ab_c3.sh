# C3 A/B on one box (tuning helper): wait hints, and a baseline
for r in 1 2; do
  timeout 300 python tools/c3_probe.py 28 p3,lookup_only 2>&1 | grep "^{"
  for wh in 1 2; do GX_JIT_WAIT_HINT=$wh timeout 300 python tools/c3_probe.py 28 p3 2>&1 | grep "^{" | sed "s/\"p3\"/\"p3_waithint$wh\"/"; done
done
python tools/time_configs.py C2:28 C4:28 C5:26 2>&1 | grep "^{" | cut -c1-100
