# persistent two-level rebuild: bulk (TMA) stores (default build) vs 16-B stores (s2thr)
out=gpurun_out/r02zs
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for v in base s2thr; do
  lib=""; [ $v != base ] && lib=paper_2310_05205_b200/ab/libgear_$v.so
  env ${lib:+GEAR_LIB=$lib} timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_stress.py tests/test_gpu_parity.py -q -x > $out/pytest_$v.log 2>&1; echo "pytest $v exit $? $(tail -1 $out/pytest_$v.log)"
done
for n in 5000000 10000000 20000000 40000000; do
  for rep in 1 2; do
  for v in base s2thr; do
    lib=""; [ $v != base ] && lib=paper_2310_05205_b200/ab/libgear_$v.so
    env ${lib:+GEAR_LIB=$lib} timeout 300 python tools/scan_bench.py $n 20 levels2 > $out/scan_${v}_${n}_$rep.json 2>&1; echo "$v $n $(cat $out/scan_${v}_${n}_$rep.json)"
  done
  done
done
for v in base s2thr; do
  lib=""; [ $v != base ] && lib=paper_2310_05205_b200/ab/libgear_$v.so
  for n in 10000000 40000000; do
  env ${lib:+GEAR_LIB=$lib} timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan2p --csv --log-file $out/ncu_${v}_$n.csv python tools/scan_bench.py $n 5 levels2 > /dev/null 2>&1; echo "ncu $v $n $?"
  done
done
