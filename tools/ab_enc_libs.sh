# A/B of uq_encode across prebuilt libraries (measurement only):
#   bash tools/ab_enc_libs.sh NAME=path/to/lib.so ...   (c5 fp16 rows, then c2 f32 rows)
for r in 1 2 3; do
  for kv in "$@"; do
    n=${kv%%=*}; l=${kv#*=}
    echo "$n $(UQ_LIB_AB=$PWD/$l python tools/enc_one.py c5 float16 768 384 8000000 6 | sort -t: -k2 -n | head -1)"
  done
done
