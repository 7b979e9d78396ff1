# cfg3 ADMM iteration breakdown: launch list of 3 iterations + one ncu --set full capture of the
# matvec row-product program (rnsx_kernel<Cfg<144,...>> in kRxProg mode), -k filter so cuSOLVER
# kernels are never replayed (the r01 cfg5 capture crashed on trsm)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches_admm.csv python tools/probe_admm_iter.py 3 > /dev/null 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rnsx_kernel --launch-skip 11 -c 1 \
    -o gpurun_out/r02_matvec_cfg3 python tools/probe_admm_iter.py 3 > gpurun_out/r02_ncu_matvec.log 2>&1
echo "ncu rc=$?"
