# per-tile look-back: one-barrier resolve (default build) vs the two-barrier one (oldres)
out=gpurun_out/r02res
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_stress.py -q -x > $out/pytest.log 2>&1; echo "pytest $? $(tail -1 $out/pytest.log)"
for n in 10000000 20000000 40000000; do
  for rep in 1 2 3; do
  for v in base oldres; do
    lib=""; [ $v != base ] && lib=paper_2310_05205_b200/ab/libgear_$v.so
    env ${lib:+GEAR_LIB=$lib} timeout 300 python tools/scan_bench.py $n 20 levels1_tile > $out/scan_${v}_${n}_$rep.json 2>&1; echo "$v $n $(cat $out/scan_${v}_${n}_$rep.json)"
  done; done
done
