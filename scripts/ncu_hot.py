"""Hottest straight-line SASS blocks of one kernel in an ncu report (development aid).
usage: ncu_hot.py REPORT KERNEL_REGEX [N]"""
import collections, csv, io, re, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
nshow = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sec = next((starts[q], starts[q + 1]) for q in range(len(starts) - 1) if re.search(kre, rows[starts[q]][1]))
rows = rows[sec[0]:sec[1]]
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr, data = rows[hdr_i], [r for r in rows[hdr_i + 1:] if len(r) > 5]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
tot = sum(float(r[ie] or 0) for r in data)
print(f"{rows[0][1] if len(rows[0]) > 1 else ''}: {tot:.0f} warp instructions")
op = lambda s: (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0] if s else ""
h = collections.Counter()
for r in data:
    h[op(r[src])] += float(r[ie] or 0)
print("  ", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in h.most_common(14)))
blocks, cur = [], None
for i, r in enumerate(data):
    c = float(r[ie] or 0)
    if cur and abs(cur[0] - c) < 1e-6:
        cur[2].append(r[src])
    else:
        cur = [c, i, [r[src]]]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[0] * len(b[2]))
for c, i, ss in blocks[:nshow]:
    ops = collections.Counter(op(s) for s in ss)
    print(f"  @{i:5d} count {c:10.0f} x {len(ss):3d} = {c * len(ss) / tot * 100:4.1f}%  {dict(ops.most_common(10))}")
