cd /root/repo
nvcc -o /tmp/mc_selftest scripts/mc_selftest.cu -lcuda -Wno-deprecated-gpu-targets && /tmp/mc_selftest > gpurun_out/mc_selftest.txt 2>&1; echo "mc rc=$?"; cat gpurun_out/mc_selftest.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for l in 1 16; do STRAGGLAR_OP_LANES=$l N=8 SIGMA=3 DTYPE=bfloat16 COUNT=524288 timeout 120 python scripts/trace_small.py > gpurun_out/trace_c5_l$l.json 2>&1; echo "trace rc=$?"; done
