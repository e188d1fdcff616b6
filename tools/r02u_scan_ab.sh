out=gpurun_out/r02u
mkdir -p $out
for n in 10000000 20000000; do
  timeout 300 python tools/scan_bench.py $n 20 > $out/scan_default_$n.json 2>&1; cat $out/scan_default_$n.json
  for v in cl2 c1x6 c1x6l2; do
    GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 300 python tools/scan_bench.py $n 20 levels1_chunk > $out/scan_${v}_$n.json 2>&1; echo "$v $n"; cat $out/scan_${v}_$n.json
  done
done
for n in 10000000 40000000; do
  GEAR_LIB=paper_2310_05205_b200/ab/libgear_tl.so timeout 300 python tools/scan_tl.py $n > $out/tl_$n.txt 2>&1; cat $out/tl_$n.txt
done
for v in cl2 c1x6l2; do
GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:scan_chunk --csv --log-file $out/ncu_${v}_10M.csv \
    python tools/scan_bench.py 10000000 5 levels1_chunk > /dev/null 2>&1; echo "ncu $v $?"
done
