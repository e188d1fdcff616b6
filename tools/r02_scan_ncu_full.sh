# ncu --set full captures of the final CDF kernels at 10 M keys: the chunked
# look-back (scan_chunk_kernel), the per-tile look-back (scan_kernel, at 40 M
# where it is auto-selected) and the persistent two-level rebuild (scan2p_kernel)
out=gpurun_out/r02_scanfull
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_chunk -s 2 -c 1 \
  -o $out/scan_chunk_10M_full python tools/scan_bench.py 10000000 3 levels1_chunk > $out/ncu_chunk.log 2>&1; echo "chunk $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan2p -s 2 -c 1 \
  -o $out/scan2p_10M_full python tools/scan_bench.py 10000000 3 levels2 > $out/ncu_s2p.log 2>&1; echo "s2p $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_kernel" -s 2 -c 1 \
  -o $out/scan_tile_40M_full python tools/scan_bench.py 40000000 3 levels1_tile > $out/ncu_tile.log 2>&1; echo "tile $?"
