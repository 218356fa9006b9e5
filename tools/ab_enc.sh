# A/B of uq_encode between libuq.so and $AB (default libuq_ab.so): c5 fp16 rows (and f32 c2 rows)
AB=${AB:-$PWD/paper_2506_00528_b200/libuq_ab.so}
for i in 1 2; do
  echo "A $(python tools/enc_one.py c5 float16 768 384 8000000 6 | tail -1)"
  echo "B $(UQ_LIB_AB=$AB python tools/enc_one.py c5 float16 768 384 8000000 6 | tail -1)"
  echo "A $(python tools/enc_one.py c2 float32 768 384 2000000 6 | tail -1)"
  echo "B $(UQ_LIB_AB=$AB python tools/enc_one.py c2 float32 768 384 2000000 6 | tail -1)"
done
