# e2e sweep of the streamed host path: compute streams x chunk ramps
run() {  # tag banks ramp
SPHBI_STREAM_BANKS=$2 SPHBI_STREAM_RAMP=$3 timeout 300 python bench.py --no-cpu-baseline --steps 8 --warmup 3 > gpurun_out/tl_$1.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/tl_$1.log').read().strip().splitlines()[-1]); print('banks $2 ramp $3: value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))"
}
for r in 1,2,3,4,3,2,1 1,2,3,3,3,3,2,1 1,2,2,3,3,3,2,2,1 1,1,2,2,3,3,2,2,1,1; do
for b in 2 3; do run x $b $r; done; done
