for tb in 128 256 512; do
  echo "== tile bytes $tb"
  SSSP_BUCKET_TILE_BYTES=$tb python tools/queue_probe.py 2>&1 | grep -E "loop K=200|k=64"
  SSSP_BUCKET_TILE_BYTES=$tb SSSP_BUCKET_TRACE=1 python tools/trace_bucket.py 2>&1 | sed -n 3,4p
done
for tb in 256 512; do
  echo "== cfg4 tile bytes $tb"
  SSSP_BUCKET_TILE_BYTES=$tb timeout 600 python tools/trace_cfg4.py 2>&1 | grep "^ms"
done
