"""A/B a config's kernels under generator / engine switches: bit-equality with the first variant and
device time per launch (CUDA events; the config's shots, or AB_SHOTS; AB_REPS launches).
    python tools/ab.py CFG "ENV=1,ENV2=3" "..."      ("" = defaults)"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2604_27058_b200.configs import CONFIGS  # noqa: E402
from paper_2604_27058_b200.engine import DeviceProgram  # noqa: E402
from paper_2604_27058_b200.program import Program  # noqa: E402

cfg = int(sys.argv[1])
variants = sys.argv[2:] or [""]
P = Program.load(f"paper_2604_27058_b200/programs/c{cfg}.npz")
shots = int(os.environ.get("AB_SHOTS", CONFIGS[cfg]["shots"]))
reps = int(os.environ.get("AB_REPS", 12))
ref = None
for v in variants:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    dp = DeviceProgram(P)
    out = dp.alloc_device_outputs(shots)
    for k in ("meas", "det", "obs", "accepted"):
        out[k].zero_()  # padding words are never written
    dp.sample_device(shots, out, seed=7)
    torch.cuda.synchronize()
    for k, o in old.items():
        if o is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = o
    got = {k: out[k].clone() for k in ("meas", "det", "obs", "accepted")}
    same = None if ref is None else all(torch.equal(got[k], ref[k]) for k in got)
    if ref is None:
        ref = got
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ms = []
    for s in range(reps):
        flush.fill_(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dp.sample_device(shots, out, seed=100 + s)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    print(json.dumps({"cfg": cfg, "variant": v or "default", "equal_to_first": same, "ms_min": ms[0],
                      "ms_med": ms[len(ms) // 2], "jit": dp.jit_status()[:60]}), flush=True)
    dp.close()
