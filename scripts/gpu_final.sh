#!/bin/bash
# Final measurement session (one GPU): GPU tests, bench lines for configs 3/4/5, the ncu launch
# list of the config-3 bench command, one ncu --set full capture of the config-3 and config-4
# kernels at steady state, CUPTI timelines.  Outputs under gpurun_out/final/.
O=gpurun_out/final
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for r in 1 2 3; do python bench.py > $O/bench_config3_$r.log 2>&1; done
python bench.py --steps 20 --warmup 5 > $O/bench_config3_20steps.log 2>&1
python bench.py --config 4 > $O/bench_config4.log 2>&1
python bench.py --config 5 > $O/bench_config5.log 2>&1
python scripts/diag_timeline.py 3 nosync > $O/timeline_config3.log 2>&1
python scripts/diag_timeline.py 4 > $O/timeline_config4.log 2>&1
python scripts/diag_ktime.py 3 F3 4f 5f > $O/ktime.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_config3_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launches.log 2>&1
python scripts/run_cfg.py --config 3 --iters 30 > $O/run_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"row_pass|prop|small_step" \
    --launch-skip 60 -c 12 -o $O/full3 python scripts/run_cfg.py --config 3 --iters 30 > $O/ncu_full3.log 2>&1
ncu -i $O/full3.ncu-rep --page raw --csv > $O/ncu_full_raw_config3.csv 2>/dev/null
python scripts/run_cfg.py --config 4 --iters 12 > $O/run_cfg4.log 2>&1 && \
ncu --set full --clock-control none -k regex:"small_step|row_solve|row_pass|incr" \
    --launch-skip 20 -c 6 -o $O/full4 python scripts/run_cfg.py --config 4 --iters 12 > $O/ncu_full4.log 2>&1
ncu -i $O/full4.ncu-rep --page raw --csv > $O/ncu_full_raw_config4.csv 2>/dev/null
rm -f $O/*.ncu-rep
echo done
