mkdir -p gpurun_out
timeout 300 python tools/e2e_loop_probe.py ising2d_32768_strang
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv -lms 200 > gpurun_out/clk.csv 2>&1 & P=$!
timeout 300 python tools/e2e_loop_probe.py ising2d_32768_strang > /dev/null
kill $P; sort gpurun_out/clk.csv | uniq -c | sort -rn | head -8
