set -x
CFGS="3" bash scripts/ab.sh
CFGS="4 2" bash scripts/ab_bench.sh
