# quick measurement set: trace, latency probe, bench (no CPU leg)
./tools/vec_trace > gpurun_out/$1_trace.txt 2>&1
python tools/stitch_latency.py 192 > gpurun_out/$1_lat.txt 2>&1
python bench.py --no-cpu --e2e-steps 10 > gpurun_out/$1_bench.json 2> gpurun_out/$1_bench.err
