#!/bin/bash
# GPU-side evidence capture for one round (run under gpurun from the repo root; gpurun brings back at
# most 64 MiB, so it runs in two parts).  Writes gpurun_out/.
#   PART=1: GPU tests, bench line, launch list of the bench command (cold-cache, serialised: compare
#           SHARES, not absolutes), `ncu --set full` of the C2 SpAdd kernels (staged + fused) and the
#           k = 3 partition kernel.
#   PART=2: `ncu --set full` of the C5 (at scale 0.25) and C3 SpMV kernels.
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
if [ "${PART:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu --no-e2e \
      > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spadd4_kernel|partition_kernel" -s 4 -c 3 \
      -o gpurun_out/full_c2 -f python profiles/run_once.py c2 --steps 3 > gpurun_out/ncu_full_c2.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spadd4_kernel|s4_place" -s 0 -c 2 \
      -o gpurun_out/full_c2_staged -f python profiles/run_staged.py > gpurun_out/ncu_full_c2_staged.log 2>&1
else
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmv3_kernel" -s 1 -c 1 \
      -o gpurun_out/full_c5 -f python profiles/run_once.py c5 --scale 0.25 --steps 2 > gpurun_out/ncu_full_c5.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spmv3_kernel" -s 1 -c 1 \
      -o gpurun_out/full_c3 -f python profiles/run_once.py c3 --steps 2 > gpurun_out/ncu_full_c3.log 2>&1
fi
# summaries on the box; the reports themselves only with KEEP_REPS=1 (gpurun returns <= 64 MiB)
for r in gpurun_out/full_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=$(basename "$r" .ncu-rep)
  python profiles/ncu_summary.py "$r" > "gpurun_out/ncu_${b}.txt" 2>&1
  python profiles/src_hot.py "$r" 60 > "gpurun_out/src_${b}.txt" 2>&1
  [ "${KEEP_REPS:-0}" = "1" ] || rm -f "$r"
done
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu.txt
