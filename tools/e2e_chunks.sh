# e2e A/B of the field copy-out schedule (HOBO_E2E_TAIL halvings, HOBO_E2E_HEAD quarter waves)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "host_entry or packed_entry or stream_k or graph or strong" 2>&1 | tail -1
for v in "${@:-1 2}"; do
set -- $v
HOBO_E2E_TAIL=$1 HOBO_E2E_HEAD=$2 timeout 300 python bench.py --steps 30 > gpurun_out/tail_$1_$2.json 2>gpurun_out/tail.err
python -c "
import json,sys; d=json.loads(open('gpurun_out/tail_$1_$2.json').read().strip().splitlines()[-1])
print('tail $1 head $2', round(d['value']/1e6,2), {k:(round(d[k]['value']/1e6,2), round(d[k]['ms_per_step'],3)) for k in ('e2e','e2e_without_fields','e2e_packed')})"
done
