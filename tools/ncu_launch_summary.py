"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (the bench command under
ncu, one row per kernel launch) into per-kernel launch counts, total time and share of the total."""
import csv
import json
import sys
from collections import OrderedDict


def main(path, out, command):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "").strip()
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[iv].replace(",", "")) / 1e6
    total = sum(v[1] for v in agg.values())
    res = {"command": command, "total_ms": total,
           "kernels": [{"kernel": k, "launches": v[0], "ms": v[1], "share": v[1] / total}
                       for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], " ".join(sys.argv[3:]))
