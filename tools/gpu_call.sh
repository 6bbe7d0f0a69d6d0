mkdir -p gpurun_out
bash tools/profile.sh ising2d_32768
