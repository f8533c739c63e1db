#!/bin/bash
# One GPU session: tests, bench, launch list, one ncu --set full of the raster kernels.
# usage: tools/gpu_round.sh TAG [tests|notests]
TAG=${1:-x}
mkdir -p gpurun_out
if [ "${2:-tests}" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_view.py > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_raster|k_project|k_onesweep|k_scan_emit" -c 16 -o gpurun_out/${TAG}_full python tools/profile_view.py > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
