# A/B of one env knob on the greedy CTC regimes: gpu_ab_env.sh VAR VAL_A VAL_B
set -e
for i in 1 2; do
  for v in "$2" "$3"; do echo "== $1=$v"; env "$1=$v" timeout 300 python scripts/ctc_regimes.py; done
done
