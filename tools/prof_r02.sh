# Round-2 evidence run (one B200): tests, smoke, bench line, launch list, --set full captures.
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.log 2>&1; tail -3 gpurun_out/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; tail -1 gpurun_out/r02_smoke.log
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 64 --warmup 3 --no-configs --no-stack --no-cpu > gpurun_out/r02_ncu_l.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ws_conv|encode_kernel" -s 4 -c 2 \
  -o gpurun_out/r02_prof_cfg3 -f python tools/prof_one.py cfg3 > gpurun_out/r02_ncu_f1.log 2>&1; echo "ncu cfg3 rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ws_conv|encode_kernel" -s 4 -c 2 \
  -o gpurun_out/r02_prof_L8 -f python tools/prof_one.py cfg5L8 > gpurun_out/r02_ncu_f2.log 2>&1; echo "ncu L8 rc $?"
