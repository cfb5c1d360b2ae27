#!/bin/bash
# DRAM bytes per launch of the secondary configurations' dominant sections at the bench's own scale
# (one step each under `ncu --metrics dram__bytes_*`), merged into profiles/traffic.json by
# profiles/traffic_merge.py.  Run under gpurun from the repo root.
set -u
mkdir -p gpurun_out
for c in c3 c4 c5; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/launches_$c.csv python profiles/run_once.py $c --steps 1 > gpurun_out/run_once_$c.log 2>&1
done
python profiles/traffic_merge.py gpurun_out/launches_c3.csv gpurun_out/launches_c4.csv gpurun_out/launches_c5.csv \
    > gpurun_out/traffic_secondary.json 2> gpurun_out/traffic_merge.err
