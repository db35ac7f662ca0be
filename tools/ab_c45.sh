t() { echo "== $1 $(env $2 python tools/time_configs.py C4:28 C5:26 2>&1 | grep '^{' | sed 's/.*"config": "\(C.\)".*"ms": \([0-9.]*\).*/\1 \2/' | tr '\n' ' ')"; }
for r in 1 2; do
  t default ""
  t stub "GX_JIT_DIAG_STUB_UPDATE=1"
  echo "== r1 $(python r1ref/tools/time_configs.py C4:28 C5:26 2>&1 | grep '^{' | sed 's/.*"config": "\(C.\)".*"ms": \([0-9.]*\).*/\1 \2/' | tr '\n' ' ')"
done
