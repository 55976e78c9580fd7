# e2e sweep of chunk ramps on the streamed host path (2 compute banks)
run() {  # tag ramp
SPHBI_STREAM_RAMP=$2 timeout 300 python bench.py --no-cpu-baseline --steps 8 --warmup 3 > gpurun_out/tl_$1.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/tl_$1.log').read().strip().splitlines()[-1]); print('ramp $2: value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))"
}
i=0
for r in 1,2,3,4,3,2,1 1,2,4,4,2,1 1,2,3,4,4,3,2,1 1,2,4,6,4,2,1 1,1,2,3,4,3,2,1,1 1,2,3,4,3,2,1; do
i=$((i+1)); run r$i $r; done
