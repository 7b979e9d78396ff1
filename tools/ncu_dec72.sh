set -x
python tools/probe_dec72.py 151552 3 > gpurun_out/r02_probe_dec.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_dec.csv python tools/probe_dec72.py 151552 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnsx_kernel -s 4 -c 1 -o gpurun_out/r02_rnsx72_dec python tools/probe_dec72.py 151552 1 > gpurun_out/r02_ncu_dec.log 2>&1
ls -la gpurun_out
