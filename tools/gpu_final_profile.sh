# Round-end evidence in one gpurun call: the GPU test suite, the default bench line, its ncu launch
# list, one full ncu capture of the dominant kernel (rnsx_kernel<72>, split CRT Enc stage 2) on the
# bench command, one of the node-factor Gram tile kernel (DMMA), and the cfg5 line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    --admm-iters 0 --admm-faithful-iters 0 --admm-collab-iters 0 --cfg4-n 0 --e2e-steps 1 > /dev/null 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rnsx_kernel --launch-skip 1 -c 1 \
    -o gpurun_out/final_rnsx72_bench python bench.py --steps 1 --warmup 1 --no-cpu-baseline --admm-iters 0 \
    --admm-faithful-iters 0 --admm-collab-iters 0 --cfg4-n 0 --e2e-steps 1 > gpurun_out/final_ncu_bench.log 2>&1
echo "ncu rnsx rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_kernel -c 1 \
    -o gpurun_out/final_factor_gram python tools/probe_factor.py 16 > gpurun_out/final_ncu_factor.log 2>&1
echo "ncu factor rc=$?"
timeout 900 python bench.py --values 65536 --cfg4-n 0 --admm-iters 0 --admm-faithful-iters 0 \
    --admm-collab-iters 0 --cfg5-iters 3 --steps 1 > gpurun_out/final_cfg5.json 2> gpurun_out/final_cfg5.err
echo "cfg5 rc=$?"
