"""A/B of the WS kernel with one (TPF_WS_SPLIT=1) or two DMMA warps per SMSP."""
import os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
for split in ("2", "1", "2"):
    env = dict(os.environ, TPF_WS_SPLIT=split)
    out = subprocess.run([sys.executable, os.path.join(here, "kernel_ab.py")], env=env, capture_output=True, text=True)
    print("split", split, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:])
