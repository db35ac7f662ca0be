# same-box bisection of C4/C5 across builds in r1ref/ (tuning helper)
for r in 1 2; do
  for d in r1ref b_b5f1170 b_b512d80 b_f538008 cur; do
    case $d in r1ref) t=r1ref/tools;; cur) t=tools;; *) t=r1ref/$d/tools;; esac
    echo "== $d $(python $t/time_configs.py C4:28 C5:26 2>&1 | grep '^{' | sed 's/.*"config": "\(C.\)".*"ms": \([0-9.]*\).*/\1 \2/' | tr '\n' ' ')"
  done
done
