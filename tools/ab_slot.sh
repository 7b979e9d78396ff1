# A/B of the W-stream ring slot size (PCB_RNSX_SLOT builds); each run under its own timeout
cp paper_2601_14980_b200/libpcb200.so /tmp/default.so
for v in default slot12288 slot16384 slot20480; do
  if [ "$v" != default ]; then cp paper_2601_14980_b200/libpcb200_$v.so paper_2601_14980_b200/libpcb200.so; fi
  echo "== $v"
  timeout 120 python tools/probe_dbg_modes.py 151552 2048 0 || echo "TIMEOUT/FAIL $v"
  cp /tmp/default.so paper_2601_14980_b200/libpcb200.so
done
