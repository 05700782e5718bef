# cfg3 per-GPU shares of strong scaling (65,536 total over 1/2/4/8 GPUs): kernel and step per call,
# with and without the stream-K schedule
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
mkdir -p gpurun_out/sk
for b in 65536 32768 16384 8192; do for sk in 1 0; do
  HOBO_SK=$sk timeout 300 python bench.py --batch $b --no-extras --steps 30 > gpurun_out/sk/b${b}_sk$sk.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sk/b${b}_sk$sk.json').read().strip().splitlines()[-1]); r=d['roofline']
print($b, 'SK=$sk', 'kernel', round(r['kernel_ms'],4), 'step', round(d['ms_per_step'],4), 'cand/s', round(d['value']/1e6,2))"
done; done
