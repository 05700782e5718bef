cd $GRAFT_REPO_ROOT
for cfg in cfg3 cfg3f cfg2; do
 for v in 0 1 0 1; do
  echo "$cfg desc=$v $(HOBO_CT_DESC=$v timeout 300 python bench.py --config $cfg --no-extras --steps 20 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["ms_per_step"],3), d["roofline"]["frac"], d["clocks"])')"
 done
done
for v in 0 1; do
  echo "cfg5 desc=$v $(HOBO_CT_DESC=$v timeout 400 python bench.py --config cfg5 --no-extras --steps 3 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["ms_per_step"],3), d["roofline"]["frac"], d["clocks"])')"
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
