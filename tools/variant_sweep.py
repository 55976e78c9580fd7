"""Time the cfg2 K4 pipeline for several prebuilt library variants (each in a
fresh process) -- used for launch-bound / code-shape sweeps."""
import subprocess
import sys

for lib in sys.argv[1:]:
    code = f"""
import sys; sys.path.insert(0, '.')
from pathlib import Path
from paper_2507_21686_b200 import _native as N
N.LIB_PATH = Path('{lib}')
import runpy; sys.argv = ['prof_eval', '--reps', '4']
runpy.run_path('tools/prof_eval.py', run_name='__main__')
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    last = [l for l in r.stdout.splitlines() if l.startswith("rep")][-1:] or [r.stderr[-300:]]
    print(lib, last[0], flush=True)
