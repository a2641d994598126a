set -u
mkdir -p gpurun_out
for c in 4 5; do timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g4_stage.txt 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "k1t or configs or folded or config4 or config5_full_size_oracle or kernel_paths or small_path or dscale" > gpurun_out/g4_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g4_parity.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "slab or sharded or peer" > gpurun_out/g4_slab.log 2>&1; echo "rc=$?" >> gpurun_out/g4_slab.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g4_bench5.json 2> gpurun_out/g4_bench5.err
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/g4_bench4.json 2> gpurun_out/g4_bench4.err
echo done
