"""Time a workload's device phases (tools/prof_target.py) for several prebuilt
library variants (tools/build_variant.sh), each in a fresh process.
  python tools/variant_time.py <workload args...> -- lib1.so lib2.so ..."""
import json
import subprocess
import sys

sep = sys.argv.index("--")
wargs, libs = sys.argv[1:sep], sys.argv[sep + 1:]
for lib in libs:
    code = f"""
import sys; sys.path.insert(0, '.')
from pathlib import Path
from paper_2507_21686_b200 import _native as N
N.LIB_PATH = Path('{lib}')
import runpy; sys.argv = ['prof_target'] + {wargs!r}
runpy.run_path('tools/prof_target.py', run_name='__main__')
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    if not rows:
        print(lib, "FAILED", r.stderr[-300:], flush=True)
        continue
    best = min(rows[1:] or rows, key=lambda x: x["ms_eval"])
    print(f"{lib}: pairs {best['pairs']} ms_pairs {best['ms_pairs']:.3f} ms_eval {best['ms_eval']:.3f}", flush=True)
