"""Build profiles/ncu_summary.json from ncu launch lists of `bench.py --steps 1 --warmup 0`.

Each input CSV comes from
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv python bench.py --config CFG --steps 1 --warmup 0 ...
The dominant kernel of the bench roofline is the mode-0 sketch pass (the first streamed
pass over the full tensor); its DRAM bytes per launch go to `traffic_bytes_per_launch`,
next to its algorithmic bytes (S * b + I_0 * l * b).

Usage: python tools/ncu_summary.py CFG=path.csv [CFG=path.csv ...]
"""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1703_09074_b200.synthetic import CONFIGS  # noqa: E402

ROOT = os.path.join(os.path.dirname(__file__), "..")
SKETCH_KERNELS = ("tc_pass_kernel<", "sketch_dmma_kernel", "tile_gemm_kernel")


def launches(path):
    lines = open(path, errors="replace").read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    iid, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    out = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        d = out.setdefault(r[iid], {"kernel": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    return list(out.values())


def main(args):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for a in args:
        name, csv_path = a.split("=", 1)
        cfg = CONFIGS[name]
        ls = launches(csv_path)
        first = next(d for d in ls if any(k in d["kernel"] for k in SKETCH_KERNELS)
                     and ("<80, 0>" in d["kernel"] or "<48, 0>" in d["kernel"] or "<32, 0>" in d["kernel"]
                          or "sketch_dmma" in d["kernel"] or "SketchLoader" in d["kernel"]))
        b = 8 if cfg.dtype.__name__ == "float64" else 4
        S = 1
        for e in cfg.shape:
            S *= e
        l = cfg.rank + cfg.oversampling
        algo = S * b + cfg.shape[0] * l * b
        summary[name] = {
            "kernel": first["kernel"][:120],
            "duration_ns": first.get("gpu__time_duration.sum"),
            "traffic_bytes_per_launch": first.get("dram__bytes_read.sum", 0) + first.get("dram__bytes_write.sum", 0),
            "algorithmic_bytes_per_launch": algo,
            "source": os.path.relpath(csv_path, ROOT),
        }
        setup = ("synth_reconstruct", "add_noise", "sum_and_sq")  # bench input generation, not the step
        tot = sum(d.get("gpu__time_duration.sum", 0) for d in ls if not any(x in d["kernel"] for x in setup))
        summary[name]["share_of_step_kernel_time"] = (first.get("gpu__time_duration.sum", 0) / tot) if tot else None
    json.dump(summary, open(path, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
