#!/bin/bash
# One-shot measurement pass on a GPU box (round 2): GPU test suite + smoke, per-launch stage times,
# bench lines of every config (config 5 = the default) and the reference arm, the ncu launch
# list of the default bench, and ncu --set full captures of the K1t launches of configs 5 and 4 and of the pressure-solve launches of config 5
# summarised on the box (the .ncu-rep files are too large to bring back). Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out /tmp/ncu
T=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
for c in 4 5; do timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/${T}_stage.txt 2>&1; done
for c in 5 4 3 2 1; do
  timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_pre_ncu.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:mode_tma -s 8 -c 6 \
  -o /tmp/ncu/full_cfg5 -f python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full5.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg5.ncu-rep --launches gpurun_out/${T}_launches_cfg5.csv --tag ${T}_ncu_cfg5 > gpurun_out/${T}_sum5.log 2>&1
cp profiles/${T}_ncu_cfg5.md profiles/${T}_ncu_cfg5.json gpurun_out/ 2>/dev/null
timeout 300 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_pre_ncu4.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mode_tma -s 8 -c 6 \
  -o /tmp/ncu/full_cfg4 -f python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full4.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_cfg4.ncu-rep --tag ${T}_ncu_cfg4 > gpurun_out/${T}_sum4.log 2>&1
cp profiles/${T}_ncu_cfg4.md profiles/${T}_ncu_cfg4.json gpurun_out/ 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mass_ -s 6 -c 3 \
  -o /tmp/ncu/full_k3 -f python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_fullk3.log 2>&1
python tools/ncu_summary.py /tmp/ncu/full_k3.ncu-rep --tag ${T}_ncu_k3_cfg5 > gpurun_out/${T}_sumk3.log 2>&1
cp profiles/${T}_ncu_k3_cfg5.md profiles/${T}_ncu_k3_cfg5.json gpurun_out/ 2>/dev/null
ncu -i /tmp/ncu/full_k3.ncu-rep --page source --csv --print-units base --print-source sass > /tmp/srck3.csv 2>/dev/null
python probes/ncu_loop.py /tmp/srck3.csv 0 > gpurun_out/${T}_k3u_stalls.txt 2>&1
timeout 300 python probes/k3_bench.py > gpurun_out/${T}_k3_bench.txt 2>&1
FDP_K3_U=0 timeout 300 python probes/k3_bench.py >> gpurun_out/${T}_k3_bench.txt 2>&1
ncu -i /tmp/ncu/full_cfg5.ncu-rep --page source --csv --print-units base --print-source sass > /tmp/src5.csv 2>/dev/null
python probes/ncu_src_top.py /tmp/src5.csv > gpurun_out/${T}_src_top_cfg5.txt 2>&1
echo done
