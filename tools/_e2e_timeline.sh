# e2e anatomy of the streamed host path: per-chunk timeline, chunk-ramp / bank sweeps
run() {  # tag banks ramp timeline
SPHBI_STREAM_BANKS=$2 SPHBI_STREAM_RAMP=$3 SPHBI_TIMELINE=$4 timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/tl_$1.log 2>&1
echo "== $1 banks=$2 ramp=$3"; grep -A10 "sphbi timeline" gpurun_out/tl_$1.log | tail -10
python -c "import json,sys; d=json.loads(open('gpurun_out/tl_$1.log').read().strip().splitlines()[-1]); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))"
}
run a 1 1,2,3,4,3,1 1
run b 2 1,2,3,3,2,1 1
for r in 1,2,3,3,2,1 1,2,3,4,3,2,1 1,2,2,2,2,2,1 1,2,3,3,3,2,1 1,1,1,1,1,1,1,1; do
for b in 2; do run x $b $r 0; done; done
python tools/pipe_sizes.py
