#!/bin/bash
# GPU-side evidence for the ESC scatter kernels (round 2): launch list of one SpGEMM + one SSSMM on C2's
# operands (cold-cache, serialised: compare SHARES) and `ncu --set full` of the expansion / contraction
# kernels; summaries made on the box (reports stay there).
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_esc.csv python profiles/dev/run_esc.py > /dev/null 2>&1
python profiles/launch_shares.py gpurun_out/launches_esc.csv > gpurun_out/launch_shares_esc.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"esc_expand_kernel|esc_contract_kernel" -c 4 \
    -o gpurun_out/full_esc -f python profiles/dev/run_esc.py > gpurun_out/ncu_full_esc.log 2>&1
for r in gpurun_out/full_esc.ncu-rep; do
  [ -f "$r" ] || continue
  python profiles/ncu_summary.py "$r" > gpurun_out/ncu_full_esc.txt 2>&1
  python profiles/src_hot.py "$r" 40 > gpurun_out/src_full_esc.txt 2>&1
  rm -f "$r"
done
