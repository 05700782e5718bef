#!/bin/bash
# A/B of the persistent energy kernels on cfg2 (HOBO_PERSIST_EXP switches parts off; the
# results of every run but exp 0 are wrong -- measurement only).  Extra env (e.g.
# HOBO_PERSIST_I8=0) passes through.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for e in ${EXPS:-0 1 2 4 8 3 15}; do
  HOBO_PERSIST_EXP=$e timeout 120 python bench.py --config cfg2 --no-extras --steps 10 > gpurun_out/exp_$e.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/exp_$e.json').read());print('exp $e', round(d['roofline']['kernel_ms']*1000,1), 'us', d['roofline']['mma_kind'])"
done
