#!/bin/bash
# One-shot measurement pass on a GPU box: ncu launch list and full captures (config-2 small-path /
# plane launches, config-4 K1 launches) summarised on the box (the .ncu-rep files are too large to
# bring back), then the bench line per config (reading the fresh traffic numbers) and the
# reference arm. Outputs under gpurun_out/. Pass "tests" as $1 to also run the GPU test suite and
# smoke().
set -u
mkdir -p gpurun_out /tmp/ncu
if [ "${1:-}" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pre_ncu.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mode_ --launch-skip 9 -c 6 \
  -o /tmp/ncu/full_cfg2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mode_contract --launch-skip 7 -c 7 \
  -o /tmp/ncu/full_cfg4 -f python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:mode_ --launch-skip 6 -c 3 \
  -o /tmp/ncu/full_cfg3 -f python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full3.log 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:mode_contract --launch-skip 9 -c 7 \
  -o /tmp/ncu/full_cfg5 -f python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full5.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg3.ncu-rep --tag r01_ncu_cfg3 > gpurun_out/sum3.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg5.ncu-rep --tag r01_ncu_cfg5 > gpurun_out/sum5.log 2>&1
cp profiles/r01_ncu_cfg3.md profiles/r01_ncu_cfg3.json profiles/r01_ncu_cfg5.md profiles/r01_ncu_cfg5.json gpurun_out/ 2>/dev/null
python tools/ncu_summary.py /tmp/ncu/full_cfg2.ncu-rep --launches gpurun_out/launches_cfg2.csv --tag r01_ncu_cfg2 > gpurun_out/sum2.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg4.ncu-rep --tag r01_ncu_cfg4 > gpurun_out/sum4.log 2>&1
cp profiles/r01_ncu_cfg2.md profiles/r01_ncu_cfg2.json profiles/r01_ncu_cfg4.md profiles/r01_ncu_cfg4.json gpurun_out/ 2>/dev/null
ncu -i /tmp/ncu/full_cfg2.ncu-rep --page source --csv --print-units base --print-source sass > /tmp/src2.csv 2>/dev/null
python probes/ncu_src_top.py /tmp/src2.csv > gpurun_out/src_top_cfg2.txt 2>&1
for c in 2 1 3 4 5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
timeout 600 python bench.py --config 3 --rt-reading literal > gpurun_out/bench_c3_literal.json 2> gpurun_out/bench_c3_literal.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
