# Final evidence of round 2 (last session): GPU tests, the default bench line (now with cfg5),
# and the ncu launch list of the cfg3 ADMM iterations (basic + collaborative) after the
# scheduling changes.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final5_pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 1200 python bench.py > gpurun_out/final5_bench.json 2> gpurun_out/final5_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pcb --csv \
    --log-file gpurun_out/final5_launches_admm.csv python bench.py --values 65536 --steps 1 --warmup 1 \
    --no-cpu-baseline --cfg4-n 0 --p4096-n 0 --cfg5-iters 0 --admm-iters 2 --admm-warmup 1 \
    --admm-faithful-iters 0 --admm-collab-iters 2 --e2e-steps 1 > /dev/null 2>&1
echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/final5_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    --admm-iters 0 --admm-faithful-iters 0 --admm-collab-iters 0 --cfg4-n 0 --p4096-n 0 --cfg5-iters 0 \
    --e2e-steps 1 > /dev/null 2>&1
echo "bench launches rc=$?"
# ncu launch list (per-launch device time, serialised) of the cfg3 ADMM line, basic + collaborative
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:rnsx|dec_|garner|update|quantize|onepmn|wide_kernel|fermat|sumzv|enc_prep|rs_|obfuscate|mod_words|status' \
    --csv --log-file gpurun_out/final5_launches_admm.csv python bench.py --values 65536 --steps 1 --warmup 1 \
    --no-cpu-baseline --cfg4-n 0 --p4096-n 0 --cfg5-iters 0 --admm-iters 2 --admm-warmup 1 \
    --admm-faithful-iters 0 --admm-collab-iters 2 --e2e-steps 1 > /dev/null 2>&1
echo "admm launches rc=$?"
