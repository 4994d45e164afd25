# Final round-2 evidence run: tools/prof_r02.sh plus the crossover sweep.
bash tools/prof_r02.sh
timeout 1500 python tools/crossover.py --out gpurun_out/r02_crossover.json > gpurun_out/crossover.log 2>&1; echo "crossover rc $?"
