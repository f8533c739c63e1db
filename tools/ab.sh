# usage: ab.sh variant... ; runs bench for each, prints value + phases
export S2D_ALLOW_OLD_LIB=1
for v in "$@"; do
  if [ $v = default ]; then unset S2D_LIB_PATH; else export S2D_LIB_PATH=$PWD/paper_2604_03092_b200/lib/$v/libsurfel2d.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_$v.log 2>&1
  echo $v $(tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); ph=d['phases_per_view']; print(d['value'], d['ms_per_step'], *[k+'='+str(ph[k]['ms']) for k in ph])")
done
