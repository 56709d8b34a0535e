cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/hint_ab
for v in ${VARS:-default st_ef ld_ef st_ef_ld_ef st_el default2}; do
  if [ "${v#default}" != "$v" ]; then L=""; else L="STRAGGLAR_LIB=$PWD/build/variants/lib_$v.so"; fi
  env $L python bench.py --no-cpu --steps ${STEPS:-20} > gpurun_out/hint_ab/$v.json 2> gpurun_out/hint_ab/$v.err
  python -c "import json;d=json.loads(open('gpurun_out/hint_ab/$v.json').read().strip().splitlines()[-1]); b=d['baselines_N3']; print('$v', 'B', d['value'], 'A', d['T_phaseA_us'], 'direct', d['direct_completion']['T_post_us'], 'fused', d['fused_call']['us'], 'ring', d['ring_us'], 'rhd', b['rhd_us'], 'bcast', b['bcast_post_us'], 'e2e', d['e2e']['value'])"
done
