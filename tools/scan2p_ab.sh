out=gpurun_out/r02k; mkdir -p $out
python __graft_entry__.py > /dev/null 2>&1
for lib in default c3b2 c2b2 c1b6; do
  if [ $lib = default ]; then L=paper_2310_05205_b200/libgear.so; else L=paper_2310_05205_b200/ab/libgear_$lib.so; fi
  for n in 10000000 40000000; do
    GEAR_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan2" -c 10 --csv --log-file $out/ncu_${lib}_$n.csv python tools/scan_bench.py $n 3 > /dev/null 2>&1
    python3 -c "
import csv
rows=list(csv.reader(open('$out/ncu_${lib}_$n.csv')))
h=None; v=[]
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h): v.append(int(r[h.index('Metric Value')].replace(',','')))
print('$lib', $n, sorted(v))"
  done
done
