"""Repeat one sample call per engine variant and compare every output word with the first run of
the first variant (a race shows up as a run that differs from the others).
    python tools/determinism.py CFG SHOTS REPS "ENV=1,ENV2=3" "..."      ("" = defaults)"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2604_27058_b200.engine import DeviceProgram  # noqa: E402
from paper_2604_27058_b200.program import Program  # noqa: E402

cfg, shots, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
variants = sys.argv[4:] or [""]
P = Program.load(f"paper_2604_27058_b200/programs/c{cfg}.npz")
ref = None
for v in variants:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    dp = DeviceProgram(P)
    for k, o in old.items():
        if o is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = o
    out = dp.alloc_device_outputs(shots)
    diffs = []
    for r in range(reps):
        for k in ("meas", "det", "obs", "accepted"):
            out[k].fill_(0)
        dp.sample_device(shots, out, seed=7)
        torch.cuda.synchronize()
        got = {k: out[k].clone() for k in ("meas", "det", "obs", "accepted")}
        if ref is None:
            ref = got
        d = {k: int((got[k] != ref[k]).sum().item()) for k in got}
        if any(d.values()):
            w = {k: torch.nonzero(got[k] != ref[k])[:4].tolist() for k in got if d[k]}
            diffs.append({"rep": r, "words": d, "where": w})
    print(json.dumps({"cfg": cfg, "variant": v or "default", "reps": reps, "runs_differing": len(diffs), "diffs": diffs[:3]}), flush=True)
    dp.close()
