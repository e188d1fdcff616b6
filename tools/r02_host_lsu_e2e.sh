# c3 e2e with host rows via LSU warps (1, default) vs bulk pipeline (0), alternating, 3 runs each
out=gpurun_out/r02hl2
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for rep in 1 2 3; do
for v in 1 0; do
  GEAR_COLLECT_HOST_LSU=$v timeout 600 python bench.py --config c3 --no-cpu-baseline > $out/c3_${v}_$rep.json 2>/dev/null
  python3 -c "import json; d=json.load(open('$out/c3_${v}_$rep.json')); r=d['roofline']; print('c3 host_lsu=$v', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'coll_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))" | tee -a $out/sweep.txt
done; done
