#!/bin/bash
# Round evidence on one B200 (run under gpurun): the default bench (every
# workload, headline last), the reference arm, two-level variant lines, the ncu
# launch list of the headline workload, and one `ncu --set full` capture of each
# dominant kernel -- each ncu command directly after the same command exited 0
# without ncu.  Output: gpurun_out/$TAG/.
set -x
TAG=${TAG:-r2}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 python bench.py > $O/bench_all.jsonl 2> $O/bench_all.err
timeout 600 python bench.py --impl reference > $O/reference.jsonl 2> $O/reference.err
timeout 600 python bench.py --workload hashtable --separate-widths --no-cpu --no-e2e > $O/bench_hashtable_separate.jsonl 2> $O/sep.err
for w in hashtable fixed4k long16g mixed; do timeout 600 python bench.py --workload $w --variant two-level --no-cpu --no-e2e > $O/bench2_$w.jsonl 2> $O/bench2_$w.err; done
C="python bench.py --workload hashtable --steps 2 --warmup 3 --no-e2e --no-cpu"
$C > $O/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_hashtable.csv $C > $O/ncu_l.log 2>&1
$C > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_short -s 3 -c 1 -o $O/kshort_dual $C > $O/ncu_ks.log 2>&1
C2="python bench.py --workload fixed4k --steps 2 --warmup 3 --no-e2e --no-cpu"
$C2 > $O/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wstring -s 3 -c 1 -o $O/kwstring_fixed4k $C2 > $O/ncu_kw.log 2>&1
C3="python bench.py --workload mixed --steps 1 --warmup 3 --no-e2e --no-cpu"
$C3 > $O/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wstring -s 3 -c 1 -o $O/kwstring_mixed $C3 > $O/ncu_kwm.log 2>&1
C4="python bench.py --workload long16g --steps 1 --warmup 3 --no-e2e --no-cpu"
$C4 > $O/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_node -s 3 -c 1 -o $O/knode $C4 > $O/ncu_kn.log 2>&1
C5="python bench.py --workload tiny --steps 2 --warmup 3 --no-e2e --no-cpu"
$C5 > $O/plain6.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_small -s 3 -c 1 -o $O/ksmall $C5 > $O/ncu_ksm.log 2>&1
echo done
