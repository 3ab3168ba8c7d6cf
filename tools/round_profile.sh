set -x
mkdir -p gpurun_out/r1
python bench.py > gpurun_out/r1/bench_hashtable.jsonl 2> gpurun_out/r1/bench_hashtable.err
for w in fixed4k long16g mixed; do timeout 600 python bench.py --workload $w > gpurun_out/r1/bench_$w.jsonl 2> gpurun_out/r1/bench_$w.err; done
for w in hashtable fixed4k long16g mixed; do timeout 600 python bench.py --workload $w --variant two-level --no-cpu > gpurun_out/r1/bench2_$w.jsonl 2> gpurun_out/r1/bench2_$w.err; done
C="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$C > gpurun_out/r1/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1/launches_hashtable.csv $C > gpurun_out/r1/ncu_l.log 2>&1
$C > gpurun_out/r1/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_short -s 2 -c 2 -o gpurun_out/r1/kshort $C > gpurun_out/r1/ncu_ks.log 2>&1
C2="python bench.py --workload fixed4k --steps 2 --warmup 1 --no-e2e --no-cpu"
$C2 > gpurun_out/r1/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wstring -s 1 -c 1 -o gpurun_out/r1/kwstring_fixed4k $C2 > gpurun_out/r1/ncu_kw.log 2>&1
C3="python bench.py --workload mixed --steps 1 --warmup 1 --no-e2e --no-cpu"
$C3 > gpurun_out/r1/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wstring -s 1 -c 1 -o gpurun_out/r1/kwstring_mixed $C3 > gpurun_out/r1/ncu_kwm.log 2>&1
C4="python bench.py --workload long16g --steps 1 --warmup 1 --no-e2e --no-cpu"
$C4 > gpurun_out/r1/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_node -s 1 -c 1 -o gpurun_out/r1/knode $C4 > gpurun_out/r1/ncu_kn.log 2>&1
echo done
