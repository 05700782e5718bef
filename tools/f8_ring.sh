# A/B of the e4m3 W ring depth (stages capped at 1, 2, or the default), cfg3 kernel time
cp paper_2407_19987_b200/csrc/kernels.cuh /tmp/k.orig
for cap in 0 2 1 0; do
  cp /tmp/k.orig paper_2407_19987_b200/csrc/kernels.cuh
  if [ $cap != 0 ]; then
    sed -i "s|                 : F8 ? min(C::MAXST, (PAIR ? 2 \* ring : ring) / (RPS \* p.L))|                 : F8 ? min($cap, (PAIR ? 2 * ring : ring) / (RPS * p.L))|" paper_2407_19987_b200/csrc/kernels.cuh
    grep -c "F8 ? min($cap," paper_2407_19987_b200/csrc/kernels.cuh
  fi
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
  for e in 0 4; do
    HOBO_KR_EXP=$e timeout 300 python bench.py --no-extras --steps 20 > gpurun_out/t.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/t.json').read().strip().splitlines()[-1]); r=d['roofline']
print('cap $cap exp $e', round(d['value']/1e6,3), 'kernel', round(r['kernel_ms'],4))"
  done
done
cp /tmp/k.orig paper_2407_19987_b200/csrc/kernels.cuh
