# bulk-copy collect kernel with 4 (default) / 6 / 8 warps per CTA: c3 (host rows on the LSU warps) and c2
out=gpurun_out/r02tt
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for v in t256; do
  GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "collect" > $out/pytest_$v.log 2>&1; echo "pytest $v $? $(tail -1 $out/pytest_$v.log)"
done
for rep in 1 2; do
for v in base t192 t256; do
  lib=""; [ $v != base ] && lib=paper_2310_05205_b200/ab/libgear_$v.so
  for c in c3 c2; do
  env ${lib:+GEAR_LIB=$lib} timeout 600 python bench.py --config $c --no-cpu-baseline > $out/${c}_${v}_$rep.json 2>/dev/null
  python3 -c "import json; d=json.load(open('$out/${c}_${v}_$rep.json')); r=d['roofline']; print('$c $v', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'coll_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))" | tee -a $out/sweep.txt
  done
done; done
