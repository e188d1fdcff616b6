# per-tile look-back scan: look-back window 512 (lp2) and status words 32 B apart (st4) vs default
out=gpurun_out/r02lb
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for v in lp2 st4; do
  GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 600 python -m pytest tests/test_gpu_scan.py -q -x > $out/pytest_$v.log 2>&1; echo "pytest $v $? $(tail -1 $out/pytest_$v.log)"
done
for n in 10000000 20000000 40000000; do
  for rep in 1 2; do
  for v in base lp2 st4; do
    lib=""; [ $v != base ] && lib=paper_2310_05205_b200/ab/libgear_$v.so
    env ${lib:+GEAR_LIB=$lib} timeout 300 python tools/scan_bench.py $n 20 levels1_tile > $out/scan_${v}_${n}_$rep.json 2>&1; echo "$v $n $(cat $out/scan_${v}_${n}_$rep.json)"
  done; done
done
