#!/bin/bash
# A/B timing of library variants built by profiles/build_variant.sh, on the
# GPU box: each variant's .so is copied over the in-tree library and
# bench.py timed (headline window + late window), two passes in alternating
# order.   usage: bash profiles/ab.sh OUT_DIR WORKLOAD variant1 variant2 ...
O=$1; W=$2; shift 2
mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
for pass in 1 2; do
  if [ $pass = 1 ]; then VS="$*"; else VS=$(echo "$*" | tr ' ' '\n' | tac | tr '\n' ' '); fi
  for v in $VS; do
    cp build/$v.so $L
    python bench.py --workload $W --no-cpu-baseline --traffic off --windows late --e2e-steps 2 \
      > $O/${v}_$pass.json 2> $O/${v}_$pass.err
    python - "$O/${v}_$pass.json" "$v" "$pass" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"{sys.argv[2]:12s} pass{sys.argv[3]} value {d['value']:9.1f}  ms {d['ms_per_step']:.4f}  late {d['windows']['late']['value']:9.1f} ({d['windows']['late']['ms_per_step']:.4f} ms)", flush=True)
PY
  done
done
cp $O/orig.so $L
