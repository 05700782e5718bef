# the GPU suite, smoke, and every BASELINE config through bench.py (round-end numbers)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3 | tee gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in ${CFGS:-cfg3 cfg2 cfg3f cfg4 cfg5}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value']/1e6,3), d['dtype'], 'kernel', round(r['kernel_ms'],3), 'frac', round(r['frac'],3), 'exec', round(r.get('frac_executed_of_hw_nominal',0),3), 'e2e', round(d['e2e']['value']/1e6,2), d['clocks'])" || tail -3 gpurun_out/bench_$c.err
done
