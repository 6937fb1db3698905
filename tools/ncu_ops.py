"""Dynamic SASS opcode histogram of one kernel from an ncu report."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
cnt = collections.Counter()
for r in rows[2:]:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    op = r[iS].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1] if " " in op else op
    op = op.split()[0].split(".")[0]
    cnt[op] += int(r[iE])
tot = sum(cnt.values())
print(f"total {tot}")
for op, c in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{op:12s} {c:12d} {100 * c / tot:5.1f}%")
