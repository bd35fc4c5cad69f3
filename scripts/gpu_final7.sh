#!/bin/bash
# Final round-2 measurement after the row-solver change: GPU tests, bench configs 3/4/5, the ncu
# launch list of the config-3 bench command, and one ncu --set full capture of the config-5 row solve.
O=gpurun_out/final7
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for r in 1 2; do timeout 300 python bench.py > $O/bench_config3_$r.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench_config3_20steps.log 2>&1
timeout 300 python bench.py --config 4 > $O/bench_config4.log 2>&1
timeout 600 python bench.py --config 5 > $O/bench_config5.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_short.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_config3_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launches.log 2>&1
timeout 300 python scripts/run_cfg.py --config 5 --iters 4 > $O/run_cfg5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"row_solve" \
    --launch-skip 2 -c 1 -o $O/full5 python scripts/run_cfg.py --config 5 --iters 4 > $O/ncu_full5.log 2>&1
ncu -i $O/full5.ncu-rep --page raw --csv > $O/ncu_full_raw_config5_rowsolve.csv 2>/dev/null
ncu -i $O/full5.ncu-rep --page details > $O/ncu_details_config5_rowsolve.txt 2>/dev/null
rm -f $O/*.ncu-rep
echo done
