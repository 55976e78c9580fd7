"""cfg4 (P3) evaluation time for several prebuilt library variants, each in a
fresh process. Usage: python tools/p3_variants.py lib1.so lib2.so ..."""
import subprocess
import sys

for lib in sys.argv[1:]:
    code = f"""
import sys; sys.path.insert(0, '.')
from pathlib import Path
from paper_2507_21686_b200 import _native as N
N.LIB_PATH = Path('{lib}')
import os, runpy; os.environ['REPS'] = '3'
runpy.run_path('tools/cfg4_time.py', run_name='__main__')
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    last = [l for l in r.stdout.splitlines() if l.startswith("cfg4")][-1:] or [r.stderr[-300:]]
    print(lib, last[0], flush=True)
