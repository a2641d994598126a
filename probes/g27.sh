timeout 300 python probes/one_apply.py 5 1 2 > gpurun_out/g27_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mass_solve -c 2 -o /tmp/k3 -f python probes/one_apply.py 5 1 2 > gpurun_out/g27_ncu.log 2>&1
python tools/ncu_summary.py /tmp/k3.ncu-rep --tag r02_ncu_k3_cfg5 > gpurun_out/g27_sum.log 2>&1
cp profiles/r02_ncu_k3_cfg5.md profiles/r02_ncu_k3_cfg5.json gpurun_out/ 2>/dev/null
ncu -i /tmp/k3.ncu-rep --page source --csv --print-units base --print-source sass > /tmp/k3src.csv 2>/dev/null
python probes/ncu_src_top.py /tmp/k3src.csv > gpurun_out/g27_src_top.txt 2>&1
ncu -i /tmp/k3.ncu-rep --page details --csv > gpurun_out/g27_details.csv 2>/dev/null
