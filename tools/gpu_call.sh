set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c1_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/c1_multigpu.log 2>&1; echo "multigpu rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c1_gpu.log 2>&1; echo "gpu rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --loopback > gpurun_out/c1_bench_loop.json 2> gpurun_out/c1_bench_loop.err; echo "loop rc=$?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --loopback --fused-exchange > gpurun_out/c1_bench_loopf.json 2> gpurun_out/c1_bench_loopf.err; echo "loopf rc=$?"
tail -3 gpurun_out/c1_multigpu.log gpurun_out/c1_gpu.log
