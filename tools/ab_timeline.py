"""A/B of library builds on the C4 batch: per-kind device time of one batch
solve for each given .so (development aid).  Usage: ab_timeline.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

for lib in sys.argv[1:]:
    env = dict(os.environ, FGMATTE_B200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "timeline.py"), "256"], env=env,
                         capture_output=True, text=True).stdout
    tot = {}
    sweeps = []
    for line in out.splitlines():
        f = line.split()
        if len(f) == 4:
            tot[f[0]] = tot.get(f[0], 0.0) + float(f[3])
            if f[0] == "sweep":
                sweeps.append(float(f[3]))
    print(lib, {k: round(v, 3) for k, v in tot.items()}, "sweeps", sweeps, flush=True)
