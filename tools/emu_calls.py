"""Run recorded device calls (tools/record_calls.py) on the CPU emulator (same control
header as the kernel, host arithmetic) with level perturbations.

    python tools/emu_calls.py   (reads profiles/calls_r02_ses_1500_128.json)
"""
import json, math, sys
sys.path.insert(0, "/root/repo")
import build
from paper_2405_09157_b200 import _native as nat, instances, meta, ses
eng = nat.Engine(build.build_emu())
rec = json.load(open("profiles/calls_r02_ses_1500_128.json"))
inst = instances.gen_ses(rec["n"], rec["d"], rec["seed"], rec["dist"])
D = ses.ses_range(inst)[0]
dev = ses.ses_device(inst, engine=eng)
spec = meta.OracleSpec(dev.cone, 3.0 * D / math.sqrt(2.0), rec["d"] + 1, dev, math.sqrt(2.0), meta.Orientation.MAX)
for k in range(0, 8):
    c = rec["calls"][k]
    st = meta.EarlyStopConfig(delta=c["delta"], patience=c["patience"], enabled=c["enabled"])
    for da in (0.0, 1e-12, -1e-12):
        r = meta.solve_ftp(spec, c["alpha"] * (1 + da), c["eps"], st, dev.progress, c["cap"])
        print(k, da, type(r).__name__, r.iterations, getattr(r, "reason", "sep"), r.best_progress, "| device", c.get("result", {}).get("iterations") if isinstance(c.get("result"), dict) else "")
