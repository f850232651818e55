set -x
O=gpurun_out/ev13; mkdir -p $O
for st in 0 1 2; do R2_R2CC_ONLY_STAGE=$st timeout 300 python tools/r2cc_stages.py 2>&1 | grep -v "^$" | tail -2 | sed "s/^/stage-only=$st /"; done
for d in 4 6; do DEAD=$d timeout 300 python tools/r2cc_stages.py 2>&1 | tail -2 | sed "s/^/dead=$d /"; done
# floor: sim 4 ranks, LL, 1 KiB..4 KiB: per-call period (events) vs kernel duration (ncu launch list)
R=$PWD
for v in r1 new; do
  d=$R; [ $v != new ] && d=$R/ab/$v
  (cd $d && timeout 300 python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 12 --dtypes bf16 > $R/$O/simfloor_$v.jsonl 2>/dev/null)
  python -c "
import json; print('$v period', [(json.loads(l)['bytes'], round(json.loads(l)['r2_ms']*1e3,1)) for l in open('$R/$O/simfloor_$v.jsonl')])"
  (cd $d && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:r2_ -c 60 --csv --log-file $R/$O/simfloor_${v}_ncu.csv python tools/sweep_sizes.py --sim-ranks 4 --ctas 4 --min-log2 10 --max-log2 10 --dtypes bf16 > /dev/null 2>&1)
  python - <<PY
import csv
rows = [r for r in csv.reader(open("$R/$O/simfloor_${v}_ncu.csv")) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
d = [float(r[14].replace(",", "")) for r in rows if "allreduce" in r[4] or "ring_kernel" in r[4]]
d = d[5:]
print("$v kernel duration (us): median", sorted(d)[len(d)//2] / (1000 if rows and rows[0][13] == "nsecond" else 1), "unit", rows[0][13] if rows else None, "n", len(d))
PY
done
