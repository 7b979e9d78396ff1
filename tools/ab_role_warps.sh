for np in 3 5 7; do echo "RW8 NPROD=$np"; PCB_RNSX_NPROD=$np python tools/probe_dbg_modes.py 151552 2048 0; done
cp paper_2601_14980_b200/libpcb200.so /tmp/rw8.so; cp paper_2601_14980_b200/libpcb200_rw4.so paper_2601_14980_b200/libpcb200.so
echo "RW4 NPROD=3"; python tools/probe_dbg_modes.py 151552 2048 0
cp /tmp/rw8.so paper_2601_14980_b200/libpcb200.so
