#!/bin/bash
# Round evidence in one gpurun call: bench lines per workload, ncu launch list of the
# default bench, one ncu --set full capture of the dominant encode/decode kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
for w in ${WORKLOADS:-c2 c1 c3 c5 c5rel c4}; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 300 python bench.py --impl reference --workload c4 --steps 2 --warmup 1 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_encode4k_sp|k_decode4k_sp" -s 2 -c 2 \
  -o gpurun_out/prof_c2_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_quantize|k_reconstruct" -c 2 \
  -o gpurun_out/prof_c2_coded python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_coded_c2.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -k "not sweep and not exhaustive" \
  > gpurun_out/memcheck_gpu.log 2>&1
exit 0
