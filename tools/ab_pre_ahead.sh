# offline r^n scheduling A/B on the cfg3 ADMM line (bench.py admm): PCB_PRE_AHEAD x PCB_PRE_PAIRS x PCB_RNSX_NP
for cfg in "1 0 0" "2 0 0" "2 1 0" "2 0 1" "2 1 1" "1 0 0" "2 1 1"; do
  set -- $cfg
  PCB_PRE_AHEAD=$1 PCB_PRE_PAIRS=$2 PCB_RNSX_NP=$3 timeout 300 python bench.py --values 65536 --cfg4-n 0 --p4096-n 0 --admm-faithful-iters 0 --admm-collab-iters 0 --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ahead=$1 pairs=$2 np=$3 admm', round(d['admm']['value'],5), d['admm']['iter_seconds'])"
done
