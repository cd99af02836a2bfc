# A/B of kernel builds: tools/ab_run.sh "base var..." "22 26" reps
set -e
VARS=${1:-"base"}; SCALES=${2:-"22"}; REPS=${3:-2}
for r in $(seq 1 $REPS); do
  for v in $VARS; do
    for sc in $SCALES; do
      ETB_LIB=paper_2009_07463_b200/lib/ab_$v.so timeout 900 python tools/root_profile.py --cold --scale $sc \
        > gpurun_out/ab${sc}_${v}_$r.log 2>&1
    done
  done
done
for v in $VARS; do
  [ "$v" = base ] && continue
  for sc in $SCALES; do
    for r in $(seq 1 $REPS); do
      echo "== $v s$sc rep $r"
      python tools/ab_levels.py gpurun_out/ab${sc}_base_$r.log gpurun_out/ab${sc}_${v}_$r.log
    done
  done
done
