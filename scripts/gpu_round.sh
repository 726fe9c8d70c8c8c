#!/bin/bash
# Round evidence in one gpurun call: bench lines per workload, reference arms,
# GPU tests + smoke, ncu launch list of the default bench (C3), ncu --set full
# captures of every stream-kernel variant (C3/C1: binary32 ABS, C2: binary32 REL,
# C5: binary64 ABS, C5rel: binary64 REL), memcheck and racecheck passes.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
for w in ${WORKLOADS:-c3 c2 c1 c5 c5rel c4}; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref_c3.err
timeout 300 python bench.py --impl reference --workload c2 --steps 3 --warmup 3 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
timeout 300 python bench.py --impl reference --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c3.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c3.log 2>&1
for w in c3 c2 c5 c5rel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_encode4k_sp|k_decode4k_sp" -s 2 -c 2 \
    -o gpurun_out/prof_${w}_full python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$w.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_quantize|k_reconstruct" -c 2 \
  -o gpurun_out/prof_c3_coded python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_coded_c3.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_stream.py tests/test_gpu_elementwise.py -q \
  -k "not exhaustive and not large and not fuzz_typed and not concurrent" > gpurun_out/memcheck_gpu.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_stream.py -q \
  -k "golden or grid or image_sizes or fuzz_multiblock or code_ranges or misaligned or unsafe" > gpurun_out/racecheck_gpu.log 2>&1
exit 0
