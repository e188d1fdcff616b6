# ncu evidence per config (SURVEY d.2): the collect kernel's duration, DRAM bytes and
# PCIe read/write bytes (the binding counter of the host-resident configs)
out=gpurun_out/r02_pcie
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed
for c in c1 c2 c3; do  # (c4 / c5: the host-RAM-sized tables do not fit next to ncu)
  timeout 900 ncu --metrics $M --clock-control none -k regex:collect -s 3 -c 3 --csv --log-file $out/ncu_collect_$c.csv \
    python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --graph 0 > $out/ncu_$c.log 2>&1; echo "$c $?"
done
