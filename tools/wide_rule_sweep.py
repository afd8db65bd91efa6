"""WIDE rule form (branchy vs branch-free) across P(migration) (development tool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("block", 1000, 1, 1e-4, 5, 200), ("block", 1000, 1, 3e-5, 5, 200), ("block", 1000, 1, 1e-5, 5, 200),
         ("tile", 200, 296, 1e-4, 3, 100), ("tile", 200, 296, 4e-4, 3, 100), ("tile", 200, 296, 1e-3, 3, 100),
         ("tile", 200, 296, 3e-3, 3, 100)]
for kern, L, reps, M, S, mcs in CASES:
    for form in ("branchy", "branchfree"):
        env = dict(os.environ, ESCG_WIDE_RULE=form, ESCG_DRAW_FORMAT="wide")
        code = ("import sys; sys.path.insert(0, %r); import tools.quick_perf as q; "
                "r = q.probe(%d, %d, %r, %d, M=%r, S=%d); "
                "import paper_2508_16639_b200 as e; eps = 2 * %r * %d * %d; "
                "print('%s L=%d reps=%d M=%g P(mig)=%%.4f %s %%.3e' %% (eps / (eps + 2), r['attempts_per_s']))"
                % (ROOT, L, mcs, kern, reps, M, S, M, L, L, kern, L, reps, M, form))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
        print(out.stdout.strip() or out.stderr.strip()[-300:], flush=True)
