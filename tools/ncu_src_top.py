"""Top source lines of an `ncu --page source --csv --print-source sass,cuda` export by warp-stall samples."""
import csv, gzip, sys

path, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
cur_file, hdr, lines = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] not in ("",):
        d = dict(zip(hdr, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        lines.append((s, int(d.get("Instructions Executed") or 0), cur_file, r[0], r[1].strip()[:110]))
tot = sum(l[0] for l in lines)
print("total samples", tot)
for s, ie, f, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {ie:9d} {f}:{ln} {src}")
