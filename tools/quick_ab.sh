#!/bin/bash
# Quick A/B session: binning/parity tests, then config-4 (and optionally config-5) bench per variant.
# usage: tools/quick_ab.sh TAG "pytest files" variant...
TAG=$1; TESTS=$2; shift 2
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -q -rf -x -p no:cacheprovider --timeout 300 --timeout_method thread > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
fi
bash tools/ab.sh "$@"
if [ -n "$AB_C5" ]; then
  export S2D_ALLOW_OLD_LIB=1
  for v in "$@"; do
    if [ $v = default ]; then unset S2D_LIB_PATH; else export S2D_LIB_PATH=$PWD/paper_2604_03092_b200/lib/$v/libsurfel2d.so; fi
    timeout 600 python bench.py --config 5 --no-cpu-baseline --steps 6 --warmup 3 > gpurun_out/bench5_$v.log 2>&1
    echo c5 $v $(tail -1 gpurun_out/bench5_$v.log | cut -c1-140)
  done
fi
