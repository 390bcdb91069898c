"""cfg3 (6.25M x 64, k=64) fit iteration time for each variants/*.so build."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "variants", "*.so"))):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "cfg3_split.py")], cwd=ROOT,
                       env=dict(os.environ, DNDC_LIB_PATH=lib), capture_output=True, text=True, timeout=600)
    print(os.path.basename(lib), "|", " | ".join((r.stdout.strip() or r.stderr.strip()[-300:]).splitlines()),
          flush=True)
