# racecheck in two parts: every kernel but the RNS core on the full probe, the RNS core on the
# smallest launches (racecheck instruments every shared-memory access of the persistent kernel)
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 7 \
    --kernel-name-exclude kns=rnsx_kernel python tools/sanitize_probe.py 64 > gpurun_out/r02_racecheck_other.txt 2>&1
echo "racecheck other kernels rc=$?" >> gpurun_out/r02_racecheck_summary.txt
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 7 \
    --kernel-name kns=rnsx_kernel python tools/sanitize_rnsx_min.py > gpurun_out/r02_racecheck_rnsx.txt 2>&1
echo "racecheck rnsx rc=$?" >> gpurun_out/r02_racecheck_summary.txt
