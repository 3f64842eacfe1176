for reps in 1 2; do echo "== reps $reps"; SSSP_BUCKET_TRACE=1 SSSP_BUCKET_REPS=$reps python tools/trace_rep.py 2>&1; done
echo "== reps 2 n=16384"; SSSP_BUCKET_TRACE=1 SSSP_BUCKET_REPS=2 python tools/trace_rep.py 16384 2>&1
