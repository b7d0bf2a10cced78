"""Fold ncu DRAM-byte launch lists into profiles/traffic.json.

Each input is the --csv log of
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
      --clock-control none -k regex:k_fused -s <preroll+warmup> -c 20
      python bench.py --workload W --variant V ...
named traffic_<W>_<V>.csv; the per-launch bytes of the timed launches are
averaged and divided by the launch's pixel count.

usage: python profiles/traffic_from_ncu.py gpurun_out/traffic_*.csv
"""
import csv
import json
import os
import re
import sys

PX = {"streams256": 256 * 640 * 480, "vga": 640 * 480, "hd1080": 1920 * 1080,
      "rows8k": 8192 * 8192}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def per_launch(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hi]
    ni, vi, ui, idi = (h.index(k) for k in ("Metric Name", "Metric Value", "Metric Unit", "ID"))
    out = {}
    for r in rows[hi + 1:]:
        if len(r) > vi:
            out.setdefault(r[idi], {})[r[ni]] = float(r[vi].replace(",", "")) * SCALE[r[ui]]
    return list(out.values())


def main(paths):
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    doc = json.load(open(dst)) if os.path.exists(dst) else {"per_px": {}}
    for p in paths:
        m = re.match(r"traffic_(\w+?)_(auto|ldg)\.csv$", os.path.basename(p))
        if not m:
            continue
        w, v = m.groups()
        ls = per_launch(p)
        n = len(ls)
        rd = sum(x["dram__bytes_read.sum"] for x in ls) / n / PX[w]
        wr = sum(x["dram__bytes_write.sum"] for x in ls) / n / PX[w]
        ms = sum(x["gpu__time_duration.sum"] for x in ls) / n * 1e3
        doc["per_px"][f"{w}:{v}"] = {"read_bytes_per_px": round(rd, 2),
                                     "write_bytes_per_px": round(wr, 2),
                                     "bytes_per_px": round(rd + wr, 2),
                                     "ncu_ms": round(ms, 4), "launches": n}
        print(w, v, doc["per_px"][f"{w}:{v}"])
    # stamp the library build the launches ran on (bench.py refuses a table
    # measured on another build)
    import hashlib

    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2110_14934_b200", "librgbdseg_b200.so")
    if os.path.exists(lib):
        doc["lib_sha256_16"] = hashlib.sha256(open(lib, "rb").read()).hexdigest()[:16]
    json.dump(doc, open(dst, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
