# A/B of the batched fp16 encoder (encode_f16_batch_kernel; measurement only).
# Build the variants HERE first (nvcc cross-compiles), then run this under gpurun:
#   python tools/ab_lib.py paper_2506_00528_b200/libuq_head.so -DUQ_ENC16_BATCH=0
#   python tools/ab_lib.py paper_2506_00528_b200/libuq_b8.so -DUQ_ENC16_BATCH=1 -DUQ_ENC16_BATCH_R=8
#   python tools/ab_lib.py paper_2506_00528_b200/libuq_b4.so -DUQ_ENC16_BATCH=1 -DUQ_ENC16_BATCH_R=4
# Parity of every encoder test on each variant, then timing (c5 d=768 and c3 d=1024 fp16 rows).
# Result (profiles/r02/ab_enc_f16_batched_dead_end.txt): parity green, 3396 (R=4) / 2244 (R=8) vs 3717 GB/s.
for v in b8 b4; do
  echo "== parity $v"; UQ_LIB_AB=$PWD/paper_2506_00528_b200/libuq_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "encode" 2>&1 | tail -3
done
SHAPES="c5 float16 768 384 8000000;c3 float16 1024 512 4000000" bash tools/ab_enc_libs.sh head=paper_2506_00528_b200/libuq_head.so b8=paper_2506_00528_b200/libuq_b8.so b4=paper_2506_00528_b200/libuq_b4.so
