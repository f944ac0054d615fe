"""Dynamic opcode mix of one kernel from an ncu report's source page (--import-source on):
executed warp-instructions per opcode, normalised by a unit count, and the stall-sample share.
Usage: python scripts/ncu_opmix.py <report.ncu-rep> <units> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
i_s, i_e = hdr.index("Source"), hdr.index("Instructions Executed")
i_w = hdr.index("Warp Stall Sampling (All Samples)")
ops, stall = collections.Counter(), collections.Counter()
tot = samples = 0
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= i_e or not r[i_e].isdigit():
        continue
    toks = r[i_s].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    n = int(r[i_e])
    ops[op] += n
    tot += n
    w = int(r[i_w]) if r[i_w].isdigit() else 0
    stall[op] += w
    samples += w
print(f"total {tot:.4g} warp-instr = {tot / units:.2f} per unit; {samples} stall samples")
for op, n in ops.most_common(top):
    print(f"  {op:12s} {n / units:7.2f}   samples {stall[op] / max(samples, 1):6.1%}")
