"""Group an ncu report's SASS by execution count (basic blocks) with opcode mix
and stall reasons: python tools/sass_blocks.py report.ncu-rep [kernel-regex] [units]."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
units = float(sys.argv[3]) if len(sys.argv) > 3 else 33554432
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kre:
    cmd += ["-k", f"regex:{kre}"]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
h = rows[starts[0] + 1]  # first matching kernel only
data = [r for r in rows[starts[0] + 2:starts[1]] if len(r) == len(h)]
ie, src, ss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
reasons = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_math", "stall_barrier", "stall_branch_resolving",
           "stall_dispatch", "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected", "stall_lg"]
idx = {x: h.index(x) for x in reasons}
tot = sum(float(r[ie] or 0) for r in data)
tots = sum(float(r[ss] or 0) for r in data)
print(f"warp-instr {tot:.4g}  per unit {tot / units:.2f}")
blk = collections.defaultdict(lambda: [0, 0.0, 0.0, collections.Counter(), collections.Counter()])
for r in data:
    c = float(r[ie] or 0)
    t = r[src].split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    b = blk[c]
    b[0] += 1
    b[1] += c
    b[2] += float(r[ss] or 0)
    b[3][o] += 1
    for x in reasons:
        b[4][x] += float(r[idx[x]] or 0)
print(f"{'exec':>10s} {'n':>4s} {'%ins':>5s} {'%stl':>5s}  " + " ".join(f"{x[6:11]:>5s}" for x in reasons) + "  ops")
for c, (n, ins, st, ops, rs) in sorted(blk.items(), key=lambda t: -t[1][1])[:14]:
    print(f"{c:10.0f} {n:4d} {ins / tot * 100:5.1f} {st / tots * 100:5.1f}  "
          + " ".join(f"{rs[x] / tots * 100:5.1f}" for x in reasons) + "  " + str(dict(ops.most_common(6))))
