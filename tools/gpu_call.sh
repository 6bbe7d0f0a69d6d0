python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_parity.py -q -x -k "odiff or loopback or uneven or zgb" > gpurun_out/c2_tests.log 2>&1; echo "tests rc=$?"
tail -n 3 gpurun_out/c2_tests.log
