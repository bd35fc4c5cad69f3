#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list, ncu full capture of the top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_launches.log 2>&1
# steady-state launches (the first iterations run the eigen-solver cold and the increments on the
# CUDA cores): skip 12 iterations' worth of launches of config 3
ncu --set full --clock-control none --import-source on -k regex:"row_pass|incr|reduce|small_step" \
    --launch-skip 60 -c 10 -o gpurun_out/full python scripts/run_cfg.py --config 3 --iters 30 \
    > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/full.ncu-rep --page raw --csv > gpurun_out/full_raw.csv 2>/dev/null
echo done
