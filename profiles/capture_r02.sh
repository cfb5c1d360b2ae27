#!/bin/bash
# GPU-side evidence capture, round 2 (run under gpurun from the repo root; writes gpurun_out/).
#   launch list of the bench command (cold-cache, serialised: compare SHARES, not absolutes),
#   `ncu --set full` of the C2 kernels (spadd7 + partition) and of the C2 intersection kernels,
#   summaries made on the box (the reports stay there: gpurun returns <= 64 MiB).
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --quick --no-cpu --no-e2e \
    > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spadd7_kernel|partition_kernel" -s 4 -c 2 \
    -o gpurun_out/full_c2 -f python profiles/run_once.py c2 --steps 4 > gpurun_out/ncu_full_c2.log 2>&1
for r in gpurun_out/full_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=$(basename "$r" .ncu-rep)
  python profiles/ncu_summary.py "$r" > "gpurun_out/ncu_${b}.txt" 2>&1
  python profiles/src_hot.py "$r" 60 > "gpurun_out/src_${b}.txt" 2>&1
  python profiles/ncu_summary.py "$r" --traffic > "gpurun_out/traffic_${b}.json" 2>&1
  rm -f "$r"
done
python profiles/launch_shares.py gpurun_out/launches_bench.csv > gpurun_out/launch_shares.txt 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
