# One gpurun call: the default bench line, then the ncu launch list and one full capture of the
# dominant kernel on the bench command itself (stage 2 of the split CRT Enc, rnsx_kernel<72>).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --admm-iters 0 --cfg4-n 0 --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnsx_kernel --launch-skip 1 -c 1 \
    -o gpurun_out/r02_rnsx72_bench python bench.py --steps 1 --warmup 1 --no-cpu-baseline --admm-iters 0 \
    --cfg4-n 0 --e2e-steps 1 > gpurun_out/r02_ncu_bench.log 2>&1
ls -la gpurun_out
bash tools/gpu_admm_profile.sh
