# A/B timing of two builds of libsf (build/ab/libsf_A.so vs libsf_B.so), interleaved
# A B A B on the same box: python scripts/tune.py per config, stencil launch time.
set -x
mkdir -p gpurun_out
CFGS=${CFGS:-"1 3"}
for rep in 1 2; do for v in A B; do for c in $CFGS; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > gpurun_out/ab_${v}_c${c}_$rep.log 2>&1
echo "$v c$c rep$rep $(grep -v BEST gpurun_out/ab_${v}_c${c}_$rep.log | tail -1)"
done; done; done
