# A/B kernel timing of two library builds: scripts/ab.sh WORKLOAD REPS libA libB ...
w=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for lib in "$@"; do
    printf "%s " "$lib"
    GEBQ_B200_LIB=$lib python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(' '.join(f'{n} {v[\"ms\"]*1e3:.1f}us' for n, v in k.items()), 'violations', d['violations'])"
  done
done
