"""profiles/ncu_traffic.json from an ncu CSV of dram__bytes_{read,write}.sum per launch.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none -k regex:<kernel> --csv --log-file X.csv python bench.py ...
    python tools/ncu_traffic.py X.csv profiles/ncu_traffic.json [label] [workload]

Per kernel: mean DRAM bytes (read + write) per launch over the captured launches --
the `traffic` field of bench.py's roofline object."""
import collections
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(src)
    workload = sys.argv[4] if len(sys.argv) > 4 else None  # keys "<workload>/<kernel>" (bench.py)
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, ii, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(h) or not r[mi].startswith("dram__bytes"):
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        per[r[ii]][r[mi]] += v
        names[r[ii]] = r[ki].split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    byk = collections.defaultdict(list)
    for lid, m in per.items():
        byk[names[lid]].append(sum(m.values()))
    for k, v in byk.items():
        out[f"{workload}/{k}" if workload else k] = {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v),
                                                     "source": label}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
