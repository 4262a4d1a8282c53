for v in "512 1" "1024 1" "512 2" "256 4" "128 1"; do set -- $v; echo "tpb $1 bps $2: $(SF_INTERP_TPB=$1 SF_INTERP_BPS=$2 python scripts/_rec_cost.py 2>&1 | grep -v gpurun | tr '\n' ' ')"; done
