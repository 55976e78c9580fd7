# e2e (pinned host buffers) vs the streamed path's chunk size
for L in 17 18 19 20 21; do
  SPHBI_STREAM_CHUNK_LOG2=$L timeout 300 python bench.py --no-cpu-baseline > gpurun_out/e2e_L$L.log 2>&1
  python - "$L" <<'PY'
import json, sys
L = sys.argv[1]
d = json.loads(open(f"gpurun_out/e2e_L{L}.log").read().strip().splitlines()[-1])
print(L, "value %.4g e2e %.4g" % (d["value"], d["e2e"]["value"]))
PY
done
