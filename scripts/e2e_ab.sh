# e2e A/B of run-time switches: the cfg4 line (device, single-call and pipelined e2e) and the cfg5
# line under each setting of ENVS (';'-separated, e.g. ENVS="X=1;X=2"), REPS times, alternating.
# SKIP4=1 / SKIP5=1 leave out a workload. Usage: ENVS="A=1;A=2" TAG=t bash scripts/e2e_ab.sh
mkdir -p gpurun_out
TAG=${TAG:-e2e}
out=gpurun_out/e2e_ab_${TAG}.log
: > $out
IFS=';' read -ra V <<< "${ENVS:-X=0}"
for rep in $(seq 1 ${REPS:-2}); do
  for envs in "${V[@]}"; do
    echo "== $envs" >> $out
    [ -z "$SKIP4" ] && env $envs timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sweep --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('cfg4 dev_ms %.4f e2e_pipelined_ms %.3f single_ms %.3f cold_ms %.2f' % (d['ms_per_step'], e['pipelined']['ms_per_build'], e['single_call']['build_ms'], e['single_call']['cold_ms']))" >> $out
    [ -z "$SKIP5" ] && env $envs timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5 dev_ms %.3f e2e_ms %.2f two_calls_ms %.2f' % (d['ms_per_step'], d['config']['build_ms_e2e'], d['config']['build_ms_e2e_two_calls']))" >> $out
  done
done
echo done >> $out
