"""Per-opcode and top-instruction warp-stall samples of one kernel from an
ncu report (source page, SASS). usage: ncu_source.py rep.ncu-rep <kernel regex> [skip]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
data = rows[2:]
i_src = hdr.index("Source")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_n = hdr.index("Instructions Executed")
val = lambda r, i: int(r[i]) if i < len(r) and r[i].isdigit() else 0
tot = sum(val(r, i_s) for r in data)
agg, cnt, ex = collections.Counter(), collections.Counter(), collections.Counter()
for r in data:
    if len(r) <= i_src:
        continue
    t = r[i_src].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    agg[op] += val(r, i_s)
    cnt[op] += 1
    ex[op] += val(r, i_n)
print("samples", tot, " warp-instructions executed", sum(ex.values()))
for op, v in agg.most_common(16):
    print("%-8s stall %5.1f%%  static %4d  executed %9d" % (op, 100 * v / max(tot, 1), cnt[op], ex[op]))
print("-- top instructions")
for r in sorted(data, key=lambda r: -val(r, i_s))[:int(sys.argv[4]) if len(sys.argv) > 4 else 20]:
    print("%5d  %s" % (val(r, i_s), r[i_src].strip()[:100]))
