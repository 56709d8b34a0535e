cd /root/repo
SUBS=1,8,16 ITERS=15 timeout 600 python scripts/sub_ab.py > gpurun_out/sub_ab2.jsonl 2>&1
for tb in 65536 98304 131072 196608; do
  STRAGGLAR_SUBSLICE_BYTES=$tb SUBS=16 ITERS=15 timeout 600 python scripts/sub_ab.py | sed "s/^{/{\"target\": $tb, /" >> gpurun_out/sub_ab2.jsonl 2>&1
done
