#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench lines for every
# workload (tree and two-level), the ncu launch list of the default bench, and
# one `ncu --set full` capture of each dominant kernel, each after the same
# command exited 0 without ncu.  Output: gpurun_out/$TAG/.
set -x
TAG=${TAG:-r1}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python bench.py > $O/bench_hashtable.jsonl 2> $O/bench_hashtable.err
timeout 600 python bench.py --separate-widths --no-cpu > $O/bench_hashtable_separate.jsonl 2> $O/bench_hashtable_separate.err
for w in fixed4k long16g mixed; do timeout 900 python bench.py --workload $w > $O/bench_$w.jsonl 2> $O/bench_$w.err; done
for w in hashtable fixed4k long16g mixed; do timeout 600 python bench.py --workload $w --variant two-level --no-cpu > $O/bench2_$w.jsonl 2> $O/bench2_$w.err; done
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$C > $O/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_hashtable.csv $C > $O/ncu_l.log 2>&1
$C > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_short -s 1 -c 1 -o $O/kshort_dual $C > $O/ncu_ks.log 2>&1
C1="python bench.py --separate-widths --steps 2 --warmup 1 --no-e2e --no-cpu"
$C1 > $O/plain1b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_short -s 2 -c 2 -o $O/kshort_separate $C1 > $O/ncu_ks2.log 2>&1
C2="python bench.py --workload fixed4k --steps 2 --warmup 1 --no-e2e --no-cpu"
$C2 > $O/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wstring -s 1 -c 1 -o $O/kwstring_fixed4k $C2 > $O/ncu_kw.log 2>&1
C3="python bench.py --workload mixed --steps 1 --warmup 1 --no-e2e --no-cpu"
$C3 > $O/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wstring -s 1 -c 1 -o $O/kwstring_mixed $C3 > $O/ncu_kwm.log 2>&1
C4="python bench.py --workload long16g --steps 1 --warmup 1 --no-e2e --no-cpu"
$C4 > $O/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_node -s 1 -c 1 -o $O/knode $C4 > $O/ncu_kn.log 2>&1
echo done
