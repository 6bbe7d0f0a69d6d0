# one GPU call (round 2): build, the accuracy tests, the whole -m gpu suite, the default bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_statistics.py -q -x -k "accuracy or paper_dt" > gpurun_out/c5_stats.log 2>&1; echo "stats rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/c5_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "bench rc=$?"
tail -n 3 gpurun_out/c5_stats.log gpurun_out/c5_tests.log
