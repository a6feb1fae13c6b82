"""Per-instruction view of an `ncu --page source --csv --print-source sass`
export: shared-memory wavefronts (and excess from bank conflicts) per opcode,
and the top instructions by stall samples.
    python scripts/sass_hot.py file_sass.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def num(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError):
        return 0.0


by = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
tot = [0.0, 0.0, 0.0]
for r in data:
    op = r[ix["Source"]].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    opc = op.split(" ")[0]
    w, e, s = num(r, "L1 Wavefronts Shared"), num(r, "L1 Wavefronts Shared Excessive"), num(r, "# Samples")
    by[opc][0] += w
    by[opc][1] += e
    by[opc][2] += s
    by[opc][3] += num(r, "Instructions Executed")
    tot[0] += w; tot[1] += e; tot[2] += s
print(f"shared wavefronts {tot[0]:.4g}  excessive {tot[1]:.4g}  stall samples {tot[2]:.0f}")
for opc, (w, e, s, n) in sorted(by.items(), key=lambda x: -x[1][0])[:12]:
    if w:
        print(f"  {opc:28s} wavefronts {w:12.4g} excessive {e:12.4g}  inst {n:12.4g}")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top instructions by samples:")
for r in sorted(data, key=lambda r: -num(r, "# Samples"))[:N]:
    print(f"  {num(r, '# Samples'):7.0f} {num(r, 'L1 Wavefronts Shared'):11.4g} {r[ix['Source']].strip()[:90]}")
