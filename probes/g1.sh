set -u
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 400 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g1_b4.json 2> gpurun_out/g1_b4.err
echo "b4 rc=$?"
timeout 400 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g1_plain4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1_launches_cfg4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g1_ncu_list.log 2>&1
echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mode_tma -s 6 -c 6 \
  -o /tmp/ncu/full_cfg4 -f python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g1_ncu_full4.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py /tmp/ncu/full_cfg4.ncu-rep --launches gpurun_out/g1_launches_cfg4.csv --tag r02_ncu_cfg4 > gpurun_out/g1_sum4.log 2>&1
cp profiles/r02_ncu_cfg4.md profiles/r02_ncu_cfg4.json gpurun_out/ 2>/dev/null
ncu -i /tmp/ncu/full_cfg4.ncu-rep --page source --csv --print-units base --print-source sass > /tmp/src4.csv 2>/dev/null
python probes/ncu_src_top.py /tmp/src4.csv > gpurun_out/g1_src_top_cfg4.txt 2>&1
ncu -i /tmp/ncu/full_cfg4.ncu-rep --page raw --csv --print-units base > gpurun_out/g1_raw4.csv 2>/dev/null
echo done
