mkdir -p gpurun_out
timeout 300 python bench.py --workload diff2d_8192 --no-cpu-baseline > gpurun_out/bench_diff2d_8192.log 2> gpurun_out/bench_diff2d_8192.err; tail -1 gpurun_out/bench_diff2d_8192.log > gpurun_out/bench_diff2d_8192.json
python -c "import json;d=json.load(open('gpurun_out/bench_diff2d_8192.json'));print(d['value'], d['e2e']['value'])"
