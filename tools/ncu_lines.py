"""Per CUDA source line of one ncu report: warp instructions executed and shared-memory wavefronts
(summed over the line's SASS), top N.   python tools/ncu_lines.py REP [N] [generated.cu]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
gen = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, cur, agg, text = None, None, None, {}, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0].strip():
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        text[cur] = r[1].strip()
        continue
    if cur is None:
        continue
    def num(col):
        try:
            return float(r[hdr[col]] or 0)
        except (KeyError, ValueError):
            return 0.0
    a = agg.setdefault(cur, [0.0, 0.0, 0.0])
    a[0] += num("Instructions Executed")
    a[1] += num("L1 Wavefronts Shared")
    a[2] += num("Warp Stall Sampling (All Samples)")
ti = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
ts = sum(v[2] for v in agg.values()) or 1
print(f"total: {ti:.4g} warp instructions, {tw:.4g} shared wavefronts, {ts:.4g} stall samples")
for k, v in sorted(agg.items(), key=lambda x: -(x[1][0] / ti + x[1][1] / tw))[:N]:
    t = text.get(k, "")
    if gen and k[0].endswith(".cu") and not t or t.startswith("<Unable"):
        t = gen[k[1] - 1].strip() if gen and k[1] - 1 < len(gen) else t
    print(f"{v[0]/ti*100:5.1f}% inst {v[1]/tw*100:5.1f}% smem-wf {v[2]/ts*100:5.1f}% stall  {k[0]}:{k[1]}  {t[:90]}")
