"""Device time of one cfg5 evaluation (16M particles, best of N) with a given
library variant: python tools/time_cfg5.py [lib.so] [reps]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
from paper_2507_21686_b200 import _native as N  # noqa: E402

if len(sys.argv) > 1:
    N.LIB_PATH = Path(sys.argv[1])
import bench_configs as BC  # noqa: E402
from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context  # noqa: E402

import torch  # noqa: E402

ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
sc = scenes.cfg5()
r = BC.run_device(ctx, sc, sc.kernels[0], sc.h, int(sys.argv[2]) if len(sys.argv) > 2 else 3)
print(sys.argv[1] if len(sys.argv) > 1 else "in-tree", r)
