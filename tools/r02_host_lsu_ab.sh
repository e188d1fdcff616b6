# host-resident rows by the TMA kernel's LSU warps (GEAR_COLLECT_HOST_LSU=1) vs its bulk pipeline
out=gpurun_out/r02hl
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
GEAR_COLLECT_HOST_LSU=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "host or collect or c3 or c4 or c5 or mixed" > $out/pytest_hostlsu.log 2>&1; echo "pytest exit $? $(tail -1 $out/pytest_hostlsu.log)"
for rep in 1 2; do
for v in 0 1; do
  GEAR_COLLECT_HOST_LSU=$v timeout 600 python bench.py --config c3 --no-cpu-baseline > $out/c3_${v}_$rep.json 2>/dev/null
  python3 -c "import json; d=json.load(open('$out/c3_${v}_$rep.json')); r=d['roofline']; print('c3 host_lsu=$v', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'coll_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))" | tee -a $out/sweep.txt
done; done
for v in 0 1; do
  GEAR_COLLECT_HOST_LSU=$v timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 200 > $out/c5_$v.json 2>/dev/null
  python3 -c "import json; d=json.load(open('$out/c5_$v.json')); r=d['roofline']; print('c5 host_lsu=$v', round(d['value']/1e6,4), 'e2e', round(d['e2e']['value']/1e6,4), 'coll_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3))" | tee -a $out/sweep.txt
done
