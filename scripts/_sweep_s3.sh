#!/bin/bash
# round 2 session 3: ResNet-200 batch sweep past HBM with the final kernels
mkdir -p gpurun_out/sweep_s3
python bench.py --plan resnet200_sweep_b1280_cal --incore --steps 5 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/sweep_s3/b1280_incore.json 2>/dev/null
for B in 1280 2048 3072 3584 4096; do
  python bench.py --plan resnet200_sweep_b${B}_cal --steps 5 --warmup 3 --no-cpu-baseline --no-probe > gpurun_out/sweep_s3/b${B}.json 2>/dev/null
done
ls -la gpurun_out/sweep_s3
