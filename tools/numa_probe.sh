#!/bin/bash
# Does the NUMA node of the host shard's pages change the zero-copy collect
# rate?  Topology, then c3 at N=1 with the process (and so, by first touch at
# cudaHostRegister, the pages) on each NUMA node in turn.
out=gpurun_out/numa
mkdir -p $out
{ lscpu | grep -i -E "numa|socket|model name"; nvidia-smi topo -m;
  for d in /sys/bus/pci/devices/*; do
    [ "$(cat $d/vendor 2>/dev/null)" = "0x10de" ] && [ "$(cat $d/class)" = "0x030200" ] && \
      echo "gpu $(basename $d) numa_node=$(cat $d/numa_node)"; done
  ls -d /sys/devices/system/node/node* ; } > $out/topo.txt 2>&1
cat $out/topo.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in /sys/devices/system/node/node*; do
  id=${n##*node}
  cpus=$(cat $n/cpulist)
  [ -z "$cpus" ] && continue
  taskset -c $cpus timeout 200 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > $out/c3_node$id.json
  python -c "
import json; d=json.load(open('$out/c3_node$id.json')); r=d['roofline']; print('node $id cpus $cpus', '%.2f M'%(d['value']/1e6), 'frac=%.3f'%r['frac'], 'coll_ms=%.4f'%r['avg_launch_ms'])"
done
