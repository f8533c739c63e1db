#!/bin/bash
# per-kernel GPU time of one config-4 refine iteration over 4 views for each library variant:
# tools/launches.sh TAG variant...   (variant "default" = the in-tree library)
TAG=$1; shift
mkdir -p gpurun_out
export S2D_ALLOW_OLD_LIB=1
for v in "$@"; do
  if [ $v = default ]; then unset S2D_LIB_PATH; else export S2D_LIB_PATH=$PWD/paper_2604_03092_b200/lib/$v/libsurfel2d.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_${v}_launches.csv python tools/profile_view.py > gpurun_out/${TAG}_${v}_ncu.log 2>&1
  python tools/launch_summary.py gpurun_out/${TAG}_${v}_launches.csv "$TAG $v" | tee gpurun_out/${TAG}_${v}_launches.txt
done
