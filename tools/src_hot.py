"""Per-source-line instruction counts and stall samples of an ncu report: python tools/src_hot.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, agg, samp, text = None, {}, {}, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split('/')[-1]; continue
    if len(r) < 8: continue
    try: ln = int(r[0])
    except ValueError: continue
    k = (fname, ln); text[k] = r[1].strip()[:70]
    try:
        agg[k] = agg.get(k, 0) + int(r[7] or 0); samp[k] = samp.get(k, 0) + int(r[4] or 0)
    except ValueError: pass
ti = sum(agg.values()) or 1; ts = sum(samp.values()) or 1
print(f"total warp instructions {ti}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{v/ti*100:5.1f}% inst {samp.get(k,0)/ts*100:5.1f}% stall  {k[0]}:{k[1]}  {text[k]}")
