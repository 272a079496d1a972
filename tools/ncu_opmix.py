"""Executed SASS instructions by opcode of one ncu report (source page, all files):
python tools/ncu_opmix.py REP [N] -- thread-level and warp-level counts, top N opcodes."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr, warp, thread = None, {}, {}
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < len(hdr):
        continue
    sass = r[hdr["Source"]].strip()
    if not sass:
        continue
    op = sass.split()[0]
    if op.startswith("@"):
        op = sass.split()[1]
    op = op.split(".")[0]
    try:
        warp[op] = warp.get(op, 0) + float(r[hdr["Instructions Executed"]] or 0)
        thread[op] = thread.get(op, 0) + float(r[hdr["Thread Instructions Executed"]] or 0)
    except (KeyError, ValueError):
        pass
tw = sum(warp.values()) or 1
for op, v in sorted(warp.items(), key=lambda x: -x[1])[:N]:
    print(f"{op:10s} warp {v:14.0f} ({v / tw * 100:5.1f}%)  thread {thread[op]:16.0f}")
