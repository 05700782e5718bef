# e4m3-limb path: parity tests, the headline bench, optional ncu of the headline kernel (NCU=1)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "${TESTS:-e4m3}" 2>&1 | tail -4
for v in ${RUNS:-HOBO_F8=1}; do
  env $v timeout 300 python bench.py --steps 20 --no-extras > gpurun_out/f8.json 2>gpurun_out/f8.err
  python -c "
import json; d=json.loads(open('gpurun_out/f8.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v', round(d['value']/1e6,3), 'kernel', round(r['kernel_ms'],3), 'frac', round(r['frac'],3), 'exec', round(r.get('frac_executed_of_hw_nominal',0),3), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/f8.err
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"kr_gemm" -s 4 -c 1 \
      -o gpurun_out/cfg3_f8_full -f python bench.py --config cfg3 --no-extras --steps 2 --warmup 3 > gpurun_out/ncu_full_f8.log 2>&1
tail -1 gpurun_out/ncu_full_f8.log
fi
