mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/f1_smoke.log
timeout 900 python -m pytest tests/test_gpu_fused.py -q -rf -p no:cacheprovider --timeout 300 --timeout_method thread > gpurun_out/f1_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/f1_pytest.log
for f in 1 0; do
  S2D_FUSED=$f timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/f1_bench_$f.log 2>&1
  echo fused=$f $(tail -1 gpurun_out/f1_bench_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); ph=d['phases_per_view']; print(d['value'], d['ms_per_step'], d['e2e']['value'], *[k+'='+str(ph[k]['ms']) for k in ph])")
done
