# A/B timing of the CodedArray stage (quantize / reconstruct) and the stream
# kernels of several library builds: scripts/ab_coded.sh WORKLOAD REPS libA libB ...
w=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for lib in "$@"; do
    printf "%s %s " "$w" "$(basename $lib)"
    GEBQ_B200_LIB=$lib python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; c=d['coded_stage']; print(' '.join(f'{n} {v[\"ms\"]*1e3:.1f}us' for n, v in k.items()), ' q %.1fus r %.1fus' % (c['quantize']['ms']*1e3, c['reconstruct']['ms']*1e3))"
  done
done
