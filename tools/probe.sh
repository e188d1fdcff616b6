#!/bin/bash
# Host/GPU probe for the roofline denominators.
out=gpurun_out/probe
mkdir -p $out
{ nproc; lscpu; free -g; ulimit -l; numactl -H 2>&1; nvidia-smi; nvidia-smi topo -m;
  nvidia-smi -q | grep -iE 'Link Gen|Link Width|Max|Current' | head -40; cat /proc/meminfo | head -5; } > $out/host.txt 2>&1
timeout 300 ./tools/probe > $out/probe.jsonl 2> $out/probe.err
echo "probe exit $?"
