#!/bin/bash
# ncu captures bench.py cites (roofline.traffic) and the launch lists, one config at a time:
#   bash tools/capture_r02.sh cfg3 cfg2 ...
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$c.csv \
      python bench.py --config $c --no-extras --steps 3 --warmup 3 > gpurun_out/ncu_ll_$c.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:"kr_gemm|kr_persist" -s 4 -c 1 \
      -o gpurun_out/${c}_full -f python bench.py --config $c --no-extras --steps 2 --warmup 3 > gpurun_out/ncu_full_$c.log 2>&1
  echo "$c done: $(tail -1 gpurun_out/ncu_full_$c.log)"
done
