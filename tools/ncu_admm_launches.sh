# ncu launch list (per-launch device time, serialised) of the cfg3 ADMM line, basic + collaborative
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:rnsx|dec_|garner|update|quantize|onepmn|wide_kernel|fermat|sumzv|enc_prep|rs_|obfuscate|mod_words|status' \
    --csv --log-file gpurun_out/final3_launches_admm.csv python bench.py --values 65536 --steps 1 --warmup 1 \
    --no-cpu-baseline --cfg4-n 0 --p4096-n 0 --cfg5-iters 0 --admm-iters 2 --admm-warmup 1 \
    --admm-faithful-iters 0 --admm-collab-iters 2 --e2e-steps 1 > /dev/null 2>&1
echo "admm launches rc=$?"
