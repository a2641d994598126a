#!/bin/bash
# One-shot measurement pass on a GPU box: bench lines per config, the reference arm, ncu launch
# list and full captures (config-2 small-path launches, config-4 K1) summarised on the box (the
# .ncu-rep files are too large to bring back). Outputs under gpurun_out/. Pass "tests" as $1 to
# also run the GPU test suite and smoke().
set -u
mkdir -p gpurun_out
if [ "${1:-}" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for c in 2 1 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
mkdir -p /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mode_small --launch-skip 10 -c 5 \
  -o /tmp/ncu/full_cfg2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mode_contract --launch-skip 5 -c 5 \
  -o /tmp/ncu/full_cfg4 -f python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full4.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg2.ncu-rep --launches gpurun_out/launches_cfg2.csv --tag r01_ncu_cfg2 > gpurun_out/sum2.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg4.ncu-rep --tag r01_ncu_cfg4 > gpurun_out/sum4.log 2>&1
cp profiles/r01_ncu_cfg2.md profiles/r01_ncu_cfg2.json profiles/r01_ncu_cfg4.md profiles/r01_ncu_cfg4.json gpurun_out/ 2>/dev/null
ncu -i /tmp/ncu/full_cfg2.ncu-rep --page source --csv --print-units base -k regex:mode_small 2>/dev/null | head -c 3000000 > gpurun_out/src_cfg2.csv
echo done
