#!/bin/bash
# Does the page backing of host shards (anonymous+THP vs POSIX shm) change the
# zero-copy collect rate?  c5 at N=1 both ways + the kernel's THP settings.
out=gpurun_out/host_pages
mkdir -p $out
{ cat /sys/kernel/mm/transparent_hugepage/enabled; cat /sys/kernel/mm/transparent_hugepage/shmem_enabled;
  cat /proc/meminfo | grep -i huge; mount | grep shm; } > $out/thp.txt 2>&1
cat $out/thp.txt
python __graft_entry__.py > /dev/null 2>&1
python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline | tail -1 > $out/c5_anon.json
GEAR_HOST_SHM=1 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline | tail -1 > $out/c5_shm.json
grep -h MemFree /proc/meminfo
for f in $out/c5_anon.json $out/c5_shm.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['config']['capacity'], 'frac=%.3f'%r['frac'], 'coll_ms=%.3f'%r['avg_launch_ms'])"; done
