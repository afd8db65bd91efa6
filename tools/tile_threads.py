"""Tile-kernel ensemble throughput vs CTA size (development tool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for L, reps, mcs in [(100, 1184, 300), (200, 296, 200), (400, 148, 100), (64, 2368, 300)]:
    for t in ["auto", "128", "256", "512"]:
        env = dict(os.environ)
        if t != "auto":
            env["ESCG_TILE_THREADS"] = t
        code = ("import sys; sys.path.insert(0, %r); import tools.quick_perf as q; r = q.probe(%d, %d, 'tile', %d); "
                "print(%r, r['attempts_per_s'])" % (ROOT, L, mcs, reps, "L=%d reps=%d threads=%s" % (L, reps, t)))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
        print(out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
