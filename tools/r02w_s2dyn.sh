# two-level rebuild with dynamic tile claiming (full rebuilds): parity, A/B vs static stride, timeline
out=gpurun_out/r02w
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_stress.py tests/test_gpu_parity.py -q -x > $out/pytest_scan.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest_scan.log
for n in 5000000 10000000 20000000 40000000; do
  timeout 300 python tools/scan_bench.py $n 20 levels2 > $out/scan_dyn_$n.json 2>&1; echo "dyn $n $(cat $out/scan_dyn_$n.json)"
  GEAR_LIB=paper_2310_05205_b200/ab/libgear_s2static.so timeout 300 python tools/scan_bench.py $n 20 levels2 > $out/scan_static_$n.json 2>&1; echo "static $n $(cat $out/scan_static_$n.json)"
done
SCAN_TL_RAW=$out/tl_raw_10M.txt GEAR_LIB=paper_2310_05205_b200/ab/libgear_tl.so timeout 300 python tools/scan_tl.py 10000000 > $out/tl_10M.txt 2>&1; cat $out/tl_10M.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan2p --csv --log-file $out/ncu_s2p_10M.csv python tools/scan_bench.py 10000000 5 levels2 > /dev/null 2>&1; echo "ncu $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan2p --csv --log-file $out/ncu_s2p_40M.csv python tools/scan_bench.py 40000000 5 levels2 > /dev/null 2>&1; echo "ncu $?"
