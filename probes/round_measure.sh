#!/bin/bash
# One-shot measurement pass on a GPU box: tests, bench lines per config, ncu launch list and a
# full capture of the config-2 small-path launches. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 1 3 4 5; do
  python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_v3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mode_small --launch-skip 10 -c 5 \
  -o gpurun_out/r01_full_cfg2_v3 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
