#!/bin/bash
# A/B of the int8 digit planes against the bf16 limbs on the L = 3 configs (bench.py, no extras)
cd "$(dirname "$0")/.."
for cfg in ${@:-cfg2 cfg3f cfg4 cfg5}; do
  for i8 in 1 0; do
    HOBO_I8=$i8 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-extras 2>/dev/null | tail -n 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$cfg', 'HOBO_I8=$i8', d['dtype'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'kernel_ms %.3f' % r['kernel_ms'],
      'exec %.0f' % r['executed_tflops'], 'frac_hw %.3f' % r['frac_exec_of_hw_nominal'], 'sm_mhz', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
  done
done
