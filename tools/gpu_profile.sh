#!/bin/bash
# Round profiling session (one GPU): bench lines (config 4 with the CPU baselines, config 5, the
# reference arm), an in-flight sweep, ncu launch lists (config 4 and 5) and one ncu --set full
# capture of the hot kernels.  usage: tools/gpu_profile.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 8 --warmup 3 > gpurun_out/${TAG}_c5_bench.log 2>&1; echo "c5 rc=$?"
tail -1 gpurun_out/${TAG}_c5_bench.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/${TAG}_ref.log | cut -c1-200
for f in 8 24; do
  S2D_INFLIGHT=$f timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/${TAG}_inflight$f.log 2>&1
  echo "inflight $f: $(tail -1 gpurun_out/${TAG}_inflight$f.log | cut -c1-120)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_view.py > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv "$TAG config 4" > gpurun_out/${TAG}_launches.txt
PROFILE_CONFIG=5 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_c5_launches.csv python tools/profile_view.py > gpurun_out/${TAG}_ncu_launch5.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_c5_launches.csv "$TAG config 5" > gpurun_out/${TAG}_c5_launches.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "bench launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_raster|k_project|k_onesweep|k_scan_emit|k_compact|k_tie" -c 14 -o gpurun_out/${TAG}_full \
  python tools/profile_view.py > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
cat gpurun_out/${TAG}_launches.txt gpurun_out/${TAG}_c5_launches.txt
