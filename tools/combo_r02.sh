timeout 200 python tools/probe_dbg_modes.py 151552 2048 0,2 > gpurun_out/r02_beta32.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 >> gpurun_out/r02_beta32.txt
bash tools/gpu_admm_profile.sh >> gpurun_out/r02_beta32.txt 2>&1
