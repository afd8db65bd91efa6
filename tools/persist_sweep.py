"""Per-launch vs persistent block kernel across lattice sizes (development tool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for L, mcs in [(512, 400), (1000, 400), (2000, 200), (3200, 200)]:
    for pers in ["0", "1"]:
        for k in ["1", "2", "4"]:
            env = dict(os.environ, ESCG_PERSISTENT=pers, ESCG_BLOCK_MCS=k)
            code = ("import sys; sys.path.insert(0, %r); import tools.quick_perf as q; r = q.probe(%d, %d, 'block'); "
                    "import paper_2508_16639_b200 as e; "
                    "print('L=%d persistent=%s kmax=%s', r['ctas'], r['launches'], '%%.3e' %% r['attempts_per_s'])"
                    % (ROOT, L, mcs, L, pers, k))
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
            print(out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
