for v in s3w4 s4w4 s6w4 s5w8; do
echo "== $v"
PG_LIB_VARIANT=$v PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9 | head -4
PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:"
done
