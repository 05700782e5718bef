# A/B of the e4m3 generator team count (kr_threads / NTEAM), cfg3 kernel time
cp paper_2407_19987_b200/csrc/kernels.cuh /tmp/k.orig
for tm in 4 3 2 4; do
  cp /tmp/k.orig paper_2407_19987_b200/csrc/kernels.cuh
  sed -i "s/return F8 ? kThreads + 256 : kThreads;/return F8 ? kThreads + 128 * ($tm - 2) : kThreads;/; s/constexpr int NTEAM = F8 ? 4 : 2;/constexpr int NTEAM = F8 ? $tm : 2;/" paper_2407_19987_b200/csrc/kernels.cuh
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
  timeout 300 python bench.py --no-extras --steps 20 > gpurun_out/t.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/t.json').read().strip().splitlines()[-1]); r=d['roofline']
print('teams $tm', round(d['value']/1e6,3), 'kernel', round(r['kernel_ms'],4))"
done
cp /tmp/k.orig paper_2407_19987_b200/csrc/kernels.cuh
