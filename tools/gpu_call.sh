mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/final_tests.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/final_bench.json').read().strip().splitlines()[-1])
print('value %.4g e2e %.4g frac %.3f alg %.3f clocks %s cpu %.3g launches %d' % (d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['frac_algorithmic'], d['clocks'], d['cpu_baseline']['value'], d['gpu_launches']))
r=json.loads(open('gpurun_out/final_ref.json').read().strip().splitlines()[-1]); print('ref %.4g' % r['value'])"
