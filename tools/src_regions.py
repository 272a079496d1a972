"""Instruction / stall share per source file:line range of an ncu report.
python tools/src_regions.py REP WORDS  (WORDS = 32-shot words per launch, for per-word counts)"""
import csv, io, subprocess, sys
rep = sys.argv[1]; words = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname = None; agg = {}; samp = {}; text = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path": fname = r[1].split('/')[-1]; continue
    if len(r) < 8: continue
    try: ln = int(r[0])
    except ValueError: continue
    k = (fname, ln); text[k] = r[1].strip()[:60]
    try:
        agg[k] = agg.get(k, 0) + int(r[7] or 0); samp[k] = samp.get(k, 0) + int(r[4] or 0)
    except ValueError: pass
ti = sum(agg.values()) or 1; ts = sum(samp.values()) or 1
byf = {}
for (f, l), v in agg.items():
    byf.setdefault(f, [0, 0]); byf[f][0] += v; byf[f][1] += samp.get((f, l), 0)
for f, (v, sm) in sorted(byf.items(), key=lambda x: -x[1][0]):
    print(f"{str(f):28s} {v/ti*100:5.1f}% inst {sm/ts*100:5.1f}% stall  per-word {v/words:7.1f}")
print()
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:40]:
    print(f"{v/ti*100:5.1f}% {samp.get(k,0)/ts*100:5.1f}%st {v/words:6.1f}/w  {k[0]}:{k[1]}  {text[k]}")
