# same-box A/B against the round-1 build (r1ref/, not tracked): C2, C4, C5, C1
for r in 1 2; do
  echo "== r2"; python tools/time_configs.py C2:28 C4:28 C5:26 C1:26 2>&1 | grep "^{" | cut -c1-90
  echo "== r1"; python r1ref/tools/time_configs.py C2:28 C4:28 C5:26 C1:26 2>&1 | grep "^{" | cut -c1-90
done
