"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: total time per kernel."""
import collections
import csv
import sys


def main(path, top=25):
    lines = open(path, errors="replace").read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        k = r[ik]
        k = k[:110]
        agg[k][0] += 1
        agg[k][1] += v
        order.append((k, v))
    tot = sum(v[1] for v in agg.values())
    unit = 1e6  # ns -> ms
    print(f"total kernel time {tot / unit:.2f} ms over {len(order)} launches")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[1] / unit:9.3f} ms {v[0]:6d}x  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
