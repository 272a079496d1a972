"""Host-compiler cost of the BASELINE configs: wall time of the reference
compile_circuit per config and its top cumulative functions.  Build container only (imports the
reference from /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tools/compile_profile.py [CFG ...]
"""
import cProfile
import io
import json
import pstats
import sys
import time

sys.path.insert(0, ".")
from framesim.backend import compile_circuit  # noqa: E402  (reference)

from paper_2604_27058_b200.configs import config_text  # noqa: E402

out = {}
for cfg in [int(c) for c in sys.argv[1:]] or [0, 1, 2, 3, 4]:
    text, ps = config_text(cfg)
    t0 = time.perf_counter()
    compile_circuit(text, postselect_detectors=ps)
    wall = time.perf_counter() - t0
    pr = cProfile.Profile()
    pr.enable()
    compile_circuit(text, postselect_detectors=ps)
    pr.disable()
    s = io.StringIO()
    st = pstats.Stats(pr, stream=s)
    top = []
    for (fn, line, name), (cc, nc, tt, ct, _) in sorted(st.stats.items(), key=lambda kv: -kv[1][3])[:40]:
        if "framesim" in fn:
            top.append({"fn": f"{fn.split('framesim/')[-1]}:{line}:{name}", "cum_s": round(ct, 3),
                        "self_s": round(tt, 3), "calls": nc})
    out[f"config{cfg}"] = {"compile_s": round(wall, 3), "top": top[:12]}
    print(json.dumps({f"config{cfg}": out[f"config{cfg}"]}), flush=True)
