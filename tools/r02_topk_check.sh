out=gpurun_out/r02tk
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests/test_gpu_parity.py -k topk -q -x --durations=8 > $out/pytest_topk.log 2>&1; echo "pytest topk exit $?"; tail -12 $out/pytest_topk.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k shared > $out/pytest_multi_shared.log 2>&1; echo "pytest multi shared exit $?"; tail -2 $out/pytest_multi_shared.log
timeout 900 python bench.py --strategy topk --no-cpu-baseline > $out/bench_c2_topk.json 2> $out/bench_c2_topk.err; echo "bench topk exit $?"
python tools/summarize_bench.py $out
