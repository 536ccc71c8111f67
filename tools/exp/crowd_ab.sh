# A/B: HEAD library vs the island-stream changes (never / always high priority)
run() { timeout 600 python bench.py --workload $2 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d.get('rollout',{});print('$1 $2', round(d['ms_per_step'],4), 'rollout', round(r.get('ms_per_step'),4))"; }
for rep in 1; do
cp tools/exp/lib_head.so paper_1810_05762_b200/libstampede_b200.so; run head hfh4096
cp tools/exp/lib_new.so paper_1810_05762_b200/libstampede_b200.so
STP_ISL_CROWD=1000000 run never_hi hfh4096
STP_ISL_CROWD=0 run always_hi hfh4096
STP_ISL_CROWD=24 run crowd24 hfh4096
done
