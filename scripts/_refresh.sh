#!/bin/bash
# round 2 session 3 measurement refresh (gpurun)
set -x
python bench.py > gpurun_out/s3_bench_default.json 2> gpurun_out/s3_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/s3_launches_b3072.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-probe > gpurun_out/s3_launches_bench.log 2>&1
python bench.py --plan resnet1001_2048_b2 --steps 3 --warmup 2 > gpurun_out/s3_bench_r1001.json 2> gpurun_out/s3_bench_r1001.err
python bench.py --plan gpt2p5b_b144_cal --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/s3_bench_gpt2p5b.json 2> gpurun_out/s3_bench_gpt2p5b.err
python bench.py --plan megatron8p3b_l36_b128_cal --steps 3 --warmup 2 --grad-slots 2 --no-cpu-baseline > gpurun_out/s3_bench_megatron.json 2> gpurun_out/s3_bench_megatron.err
ls -la gpurun_out/s3_*
