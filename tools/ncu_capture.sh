#!/usr/bin/env bash
# ncu --set full of the stitched main pass on the BASELINE workloads (one
# launch each), exported as CSV (details + raw metrics) into gpurun_out/; the
# .ncu-rep files stay in /tmp (size).  Plus the launch list of a short bench.
#   bash tools/ncu_capture.sh <tag>
set -u
tag=${1:-r2}
for wl in k80_n1e8 k25_n1e6 k25_n1e6_b256; do
  ncu --set full --clock-control none --import-source on -k regex:chain_fwd -c 1 -f -o /tmp/${tag}_${wl} \
      python tools/one_eval.py $wl > gpurun_out/${tag}_ncu_${wl}.log 2>&1
  ncu -i /tmp/${tag}_${wl}.ncu-rep --page details --csv > gpurun_out/${tag}_ncu_${wl}_details.csv 2>&1
  ncu -i /tmp/${tag}_${wl}.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_${wl}_raw.csv 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 3 --subconfigs "" > gpurun_out/${tag}_launch_bench.log 2>&1
