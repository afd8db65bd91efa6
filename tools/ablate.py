"""Diagnostic ablations of the block kernel (builds variants with -D flags; timings only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = {
    "base": [],
    "cheap_rng": ["ESCG_DIAG_CHEAP_RNG"],
    "no_attempts": ["ESCG_DIAG_NO_ATTEMPTS"],
    "enum_only": ["ESCG_DIAG_NO_ATTEMPTS", "ESCG_DIAG_CHEAP_RNG"],
    "no_load": ["ESCG_DIAG_NO_LOAD"],
    "no_phase_sync": ["ESCG_DIAG_NO_PHASE_SYNC"],
    "no_swap": ["ESCG_DIAG_NO_SWAP"],
}

if __name__ == "__main__":
    if sys.argv[1:2] == ["build"]:
        sys.path.insert(0, ROOT)
        from paper_2508_16639_b200.build import build
        for name, defs in VARIANTS.items():
            build(out=os.path.join(ROOT, "tools", "_ablate_%s.so" % name), defines=defs)
        sys.exit(0)
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 3200
    only = os.environ.get("ABLATE", "")
    for name in VARIANTS:
        if only and name not in only.split(","):
            continue
        env = dict(os.environ, ESCG_LIB=os.path.join(ROOT, "tools", "_ablate_%s.so" % name))
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "one_block.py"), str(L), "200"] + sys.argv[2:],
                             env=env, capture_output=True, text=True)
        print(name, out.stdout.strip(), out.stderr.strip()[-200:], flush=True)
