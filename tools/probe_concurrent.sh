#!/bin/bash
# Concurrent host-read probe: every visible GPU reads pinned host memory at the
# same time (zero-copy kernel, then DMA H2D); per-GPU and aggregate GB/s.
out=gpurun_out/probe_conc
mkdir -p $out
n=$(nvidia-smi -L | wc -l)
for mode in zc h2d; do
  for k in 1 $n; do
    for ((d=0; d<k; d++)); do ./tools/probe $mode $d 4 > $out/${mode}_k${k}_d$d.json & done
    wait
  done
done
cat $out/*.json
