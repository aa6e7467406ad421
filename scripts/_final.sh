#!/bin/bash
# round 2 session 3 final measurements (gpurun)
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/f_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
python bench.py > gpurun_out/f_bench_default.json 2> gpurun_out/f_bench_default.err
python bench.py --no-cpu-baseline > gpurun_out/f_bench_default2.json 2>/dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/f_launches_b3072.csv python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-probe > gpurun_out/f_launches.log 2>&1
python bench.py --plan resnet1001_2048_b2 --steps 3 --warmup 2 > gpurun_out/f_bench_r1001.json 2>/dev/null
python bench.py --plan gpt2p5b_b144_cal --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/f_bench_gpt2p5b.json 2>/dev/null
python bench.py --plan megatron8p3b_l36_b128_cal --steps 3 --warmup 2 --grad-slots 2 --no-cpu-baseline > gpurun_out/f_bench_megatron.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_bench_reference.json 2>/dev/null
ls -la gpurun_out/f_*
