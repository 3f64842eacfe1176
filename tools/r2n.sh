SSSP_BUCKET_TRACE=1 python tools/trace_rep.py 2>&1 | head -8
SSSP_BUCKET_TRACE=1 SSSP_BUCKET_TAGX=0 python tools/trace_rep.py 2>&1 | head -6
for e in "SSSP_BUCKET_TAGX=0" "SSSP_BUCKET_POLL=0" "SSSP_BUCKET_POLL=1" "SSSP_BUCKET_POLL=2" "SSSP_BUCKET_POLL=2 SSSP_BUCKET_POLL_NS=64" "SSSP_BUCKET_POLL=1 SSSP_BUCKET_POLL_NS=64"; do
  env $e python tools/ab_time.py 1d,2,3 40
done
