out=gpurun_out/r01x
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench exit $?"
cut -c1-400 $out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err; echo "reference exit $?"
cut -c1-300 $out/bench_reference.json
