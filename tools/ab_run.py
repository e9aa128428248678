"""Run bench.py for several library variants back to back; print per-kernel us/launch.

usage: python tools/ab_run.py TAG[,TAG...] [rounds]   (TAG 'cur' = the in-tree library)
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tags = sys.argv[1].split(",")
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 1
extra = sys.argv[3:]
for rd in range(rounds):
    for t in tags:
        env = dict(os.environ)
        if t != "cur":
            env["FLUME_B200_LIB"] = str(ROOT / "paper_2303_02346_b200" / "_ab" / t / "libflume_b200.so")
        out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "5", "--warmup", "3", "--no-cpu", *extra],
                             env=env, capture_output=True, text=True)
        try:
            j = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            print(t, "FAILED", out.stderr[-2000:])
            continue
        k = {n: round(v["us_per_launch"], 1) for n, v in j["kernels"].items()}
        print(f"{t:8s} val={j['value']:.3e} ms={j['ms_per_step']:.2f}", k, flush=True)
