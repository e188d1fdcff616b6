# chunked look-back: chunks per CTA (A/B builds), event-timed rebuilds
out=gpurun_out/r02v
mkdir -p $out
for n in 5000000 10000000 20000000 40000000; do
  for v in cpc2 cpc3 cpc4 cpc3l2; do
    GEAR_LIB=paper_2310_05205_b200/ab/libgear_$v.so timeout 300 python tools/scan_bench.py $n 20 levels1_chunk > $out/scan_${v}_$n.json 2>&1; echo "$v $n $(cat $out/scan_${v}_$n.json)"
  done
done
SCAN_TL_RAW=$out/tl_raw_cpc3_10M.txt GEAR_LIB=paper_2310_05205_b200/ab/libgear_tl.so timeout 300 python tools/scan_tl.py 10000000 > $out/tl_cpc3_10M.txt 2>&1; cat $out/tl_cpc3_10M.txt
