#!/bin/bash
# DRAM traffic of the persistent forward with / without the persisting-L2 window over its weights
# (ADPSGD_FWD_L2WIN), one bench step under ncu, then a same-box bench A/B. Output gpurun_out/<tag>_*.
tag=${1:-r02h}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for w in 0 1; do
  ADPSGD_FWD_L2WIN=$w ncu --metrics $M --clock-control none -k regex:FwdPersist -s 6 -c 6 --csv \
    --log-file gpurun_out/${tag}_l2win$w.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
    > /dev/null 2>&1
done
bash tools/ab.sh "" "ADPSGD_FWD_L2WIN=1" "" "ADPSGD_FWD_L2WIN=1" > gpurun_out/${tag}_ab.txt 2>&1
