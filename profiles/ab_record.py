"""Fold the bench lines of profiles/ab.sh runs into one experiment record of
profiles/variants_r02.json.

    python profiles/ab_record.py --name "..." --source "..." --reading "..." \
        [--adopted] [--extra extra.json] gpurun_out/r2x/ab_streams256 gpurun_out/r2x/ab_vga ...

Each directory is one workload (ab_<workload>); its <variant>_<pass>.json files
are the bench lines.  The record keeps value/late_value/ms per variant and pass.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))


def fold(d: str) -> dict:
    out: dict = {}
    for f in sorted(glob.glob(os.path.join(d, "*_[12].json"))):
        m = re.match(r"(.+)_([12])\.json$", os.path.basename(f))
        if not m:
            continue
        try:
            line = json.loads(open(f).read().strip().splitlines()[-1])
        except (IndexError, ValueError):
            out.setdefault(m.group(1), []).append(None)
            continue
        late = (line.get("windows") or {}).get("late") or {}
        out.setdefault(m.group(1), []).append({
            "value": line["value"], "ms": line["ms_per_step"],
            "late_value": late.get("value"), "late_ms": late.get("ms_per_step")})
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    ap.add_argument("--source", required=True)
    ap.add_argument("--reading", required=True)
    ap.add_argument("--adopted", action="store_true")
    ap.add_argument("--extra", help="JSON file merged into the record")
    ap.add_argument("dirs", nargs="+")
    a = ap.parse_args()
    rec = {"name": a.name, "source": a.source, "bench_mpix_s": {}}
    for d in a.dirs:
        w = os.path.basename(d.rstrip("/")).replace("ab_", "")
        rec["bench_mpix_s"][w] = fold(d)
    if a.extra:
        rec.update(json.load(open(a.extra)))
    rec["adopted"] = a.adopted
    rec["reading"] = a.reading
    path = os.path.join(HERE, "variants_r02.json")
    doc = json.load(open(path))
    doc["experiments"].append(rec)
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")
    print(json.dumps(rec["bench_mpix_s"], indent=None)[:2000])


if __name__ == "__main__":
    main()
