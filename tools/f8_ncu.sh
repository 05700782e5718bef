# ncu --set full of the e4m3 contraction at cfg3 under the given HOBO_KR_EXP (measurement switches)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for e in ${EXPS:-0}; do
HOBO_KR_EXP=$e timeout 600 ncu --set full --import-source on --clock-control none -k regex:"kr_gemm" -s 4 -c 1 \
      -o gpurun_out/cfg3_f8_exp$e -f python bench.py --config cfg3 --no-extras --steps 2 --warmup 3 > gpurun_out/ncu_f8_exp$e.log 2>&1
tail -1 gpurun_out/ncu_f8_exp$e.log
done
