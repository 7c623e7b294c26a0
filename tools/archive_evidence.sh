# Copy one evidence run (tools/evidence.sh TAG, merged into gpurun_out/) into profiles/ as the
# committed summaries.  usage: bash tools/archive_evidence.sh TAG   (run in the dev container)
cd "$(dirname "$0")/.."
T=$1; G=gpurun_out; P=profiles
tail -3 $G/ev_pytest_$T.log > $P/${T}_pytest_gpu.txt
tail -1 $G/ev_smoke_$T.log > $P/${T}_smoke.txt
grep '^{' $G/ev_bench_$T.log | tail -1 > $P/${T}_bench.jsonl
grep '^{' $G/ev_ref_$T.log | tail -1 > $P/${T}_bench_reference.jsonl
grep '^{' $G/ev_configs_$T.log > $P/${T}_configs.jsonl
grep '^{' $G/ev_hbm_$T.log > $P/${T}_hbm_ceilings.jsonl
python tools/launch_list.py $G/ev_launches_$T.csv $P/${T}_launches.csv > $P/${T}_launch_shares.txt
python tools/ncu_summary.py $G/ev_prof_$T.ncu-rep > $P/${T}_ncu_full_summary.txt
python tools/ncu_traffic.py $G/ev_prof_$T.ncu-rep $P/ncu_traffic.json > /dev/null
[ -f $G/ncu_configs_$T.jsonl ] && cp $G/ncu_configs_$T.jsonl $P/${T}_ncu_configs.jsonl
[ -f $G/l1_first_$T.txt ] && cp $G/l1_first_$T.txt $P/${T}_l1_pipe.txt
ls -la $P/${T}_*
