"""Summarise an `ncu --set full` report as markdown (for profiles/).
python tools/ncu_summary.py REPORT.ncu-rep TITLE > profiles/NAME.md"""
import csv, io, subprocess, sys

rep, title = sys.argv[1], sys.argv[2]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, units, v = raw[0], raw[1], raw[2]
m = {n: (v[i], units[i]) for i, n in enumerate(h)}


def g(name, fmt="{}"):
    if name not in m:
        return "n/a"
    val, u = m[name]
    return fmt.format(val) + (f" {u}" if u else "")


rows = [
    ("kernel", m.get("Kernel Name", ("?", ""))[0]),
    ("grid x block", f"{g('launch__grid_size')} x {g('launch__block_size')}"),
    ("duration", g("gpu__time_duration.sum")),
    ("DRAM read / write", f"{g('dram__bytes_read.sum')} / {g('dram__bytes_write.sum')}"),
    ("DRAM throughput (% of peak)", g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
    ("SM throughput (% of peak)", g("sm__throughput.avg.pct_of_peak_sustained_elapsed")),
    ("executed IPC (active)", g("sm__inst_executed.avg.per_cycle_active")),
    ("issue slots busy", g("sm__inst_issued.avg.pct_of_peak_sustained_active")),
    ("warp instructions executed", g("smsp__inst_executed.sum")),
    ("registers / thread", g("launch__registers_per_thread")),
    ("dynamic smem / block", g("launch__shared_mem_per_block_dynamic")),
    ("occupancy theoretical / achieved", f"{g('sm__maximum_warps_per_active_cycle_pct')} / {g('sm__warps_active.avg.pct_of_peak_sustained_active')}"),
    ("FP64 pipe (% of peak, active)", g("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")),
    ("ALU pipe (% of peak, active)", g("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")),
    ("shared bank conflicts", g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")),
    ("shared wavefronts", g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")),
]
stalls = []
for n, (val, u) in m.items():
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(val.replace(",", "")), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
stalls.sort(reverse=True)
print(f"# {title}\n")
print(f"Source: `{rep.split('/')[-1]}` (`ncu --set full --clock-control none --import-source on`, one launch).\n")
print("| metric | value |\n|---|---|")
for k, val in rows:
    print(f"| {k} | {val} |")
print("\nTop warp stall reasons (cycles per issued instruction):\n")
print("| reason | cycles |\n|---|---|")
for val, n in stalls[:8]:
    print(f"| {n} | {val:.2f} |")
# hottest source lines
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
fname, agg, samp, text = None, {}, {}, {}
for r in src:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = (fname, ln)
    text[key] = r[1].strip()[:90]
    try:
        agg[key] = agg.get(key, 0) + int(r[7] or 0)
        samp[key] = samp.get(key, 0) + int(r[4] or 0)
    except ValueError:
        pass
tot_s = sum(samp.values()) or 1
if samp:
    print("\nHottest source lines (share of warp-stall samples):\n")
    print("| file:line | samples | source |\n|---|---|---|")
    for key in sorted(samp, key=lambda k: -samp[k])[:12]:
        print(f"| {key[0]}:{key[1]} | {100 * samp[key] / tot_s:.1f}% | `{text[key].replace('|', '/')}` |")
