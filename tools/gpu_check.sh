#!/bin/bash
# Guarded GPU session: a 60 s smoke first (a hang there stops the session), then the GPU tests
# with a per-test timeout that kills a stuck process (thread method), then A/B benches.
# usage: tools/gpu_check.sh TAG [variant ...]
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/${TAG}_smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1500 python -m pytest tests -m gpu -q -rf -x -p no:cacheprovider --timeout 300 --timeout_method thread \
  > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
[ $# -gt 0 ] && bash tools/ab.sh "$@"
exit 0
