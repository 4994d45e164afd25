set -x
python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-stack > gpurun_out/ncu_l.log 2>&1
ncu --set full --import-source on --clock-control none -s 6 -c 2 -o gpurun_out/prof_cfg2_final -f python tools/prof_one.py cfg2 > gpurun_out/ncu_f1.log 2>&1
ncu --set full --import-source on --clock-control none -s 6 -c 2 -o gpurun_out/prof_L0_final -f python tools/prof_one.py cfg5L0 > gpurun_out/ncu_f2.log 2>&1
ncu --set full --import-source on --clock-control none -s 6 -c 2 -o gpurun_out/prof_L8_final -f python tools/prof_one.py cfg5L8 > gpurun_out/ncu_f3.log 2>&1
python tools/time_all.py > gpurun_out/time_all_final.jsonl 2>&1
echo done
ncu --set full --import-source on --clock-control none -k regex:"tc_gemm|im2col_t" -s 2 -c 2 -o gpurun_out/prof_tcL0 -f python tools/tc_one.py cfg5L0 256 > gpurun_out/ncu_tc0.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"tc_gemm|im2col_t" -s 2 -c 2 -o gpurun_out/prof_tcL8 -f python tools/tc_one.py cfg5L8 256 > gpurun_out/ncu_tc8.log 2>&1
python tools/crossover.py --out gpurun_out/r01_crossover.json > gpurun_out/xo.log 2>&1
echo done2
