# chunked look-back: phase-2 bulk (TMA) stores, immediate / deferred reloads (A/B builds)
out=gpurun_out/r02xs
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for v in cts cts2 cts2l2; do
  GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_stress.py -q -x > $out/pytest_$v.log 2>&1; echo "pytest $v exit $? $(tail -1 $out/pytest_$v.log)"
done
for n in 5000000 10000000 20000000; do
  timeout 300 python tools/scan_bench.py $n 20 levels1_chunk > $out/scan_base_$n.json 2>&1; echo "base $n $(cat $out/scan_base_$n.json)"
  for v in cts cts2 cts2l2; do
    GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 300 python tools/scan_bench.py $n 20 levels1_chunk > $out/scan_${v}_$n.json 2>&1; echo "$v $n $(cat $out/scan_${v}_$n.json)"
  done
done
SCAN_TL_RAW=$out/tl_raw_10M.txt GEAR_LIB=paper_2310_05205_b200/ab/libgear_tl.so timeout 300 python tools/scan_tl.py 10000000 > $out/tl_10M.txt 2>&1; cat $out/tl_10M.txt
