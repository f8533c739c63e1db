for k in "$@"; do
  S2D_INFLIGHT=$k timeout 600 python bench.py --no-cpu-baseline --steps 15 > gpurun_out/bench_if$k.log 2>&1
  echo inflight=$k $(tail -1 gpurun_out/bench_if$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'])")
done
