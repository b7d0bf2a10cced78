#!/bin/bash
# A/B of K1ws builds (build/<name>.so from profiles/build_variant.sh) with
# --variant ws on the given workloads; the in-tree library is restored after.
#   usage: bash profiles/ab_ws.sh OUT_DIR "streams256 vga" name1 name2 ...
O=$1; WS=$2; shift 2
mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
for v in "$@"; do for w in $WS; do
  cp build/$v.so $L
  VAR=ws; [ "$v" = "base" ] && VAR=auto
  timeout 300 python bench.py --workload $w --variant $VAR --no-cpu-baseline --traffic off --windows late --e2e-steps 2 > $O/${w}_$v.json 2> $O/${w}_$v.err
  python - "$O/${w}_$v.json" "$v" "$w" <<'PY' || tail -3 $O/${w}_$v.err
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"{sys.argv[3]:10s} {sys.argv[2]:8s} value {d['value']:9.1f}  ms {d['ms_per_step']:.4f}  late {d['windows']['late']['value']:9.1f}", flush=True)
PY
done; done
cp $O/orig.so $L
