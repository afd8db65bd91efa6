"""Block-kernel throughput vs (threads, MCS per launch) for one lattice size (development tool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
mcs = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for t in ["512", "640"]:
    for k in ["1", "2", "3", "4"]:
        env = dict(os.environ, ESCG_BLOCK_THREADS=t, ESCG_BLOCK_MCS=k)
        code = ("import sys; sys.path.insert(0, %r); import tools.quick_perf as q; r = q.probe(%d, %d, 'block'); "
                "print('threads=%s kmax=%s', r['ctas'], r['launches'], '%%.3e' %% r['attempts_per_s'])" % (ROOT, L, mcs, t, k))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
        print(out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
