# A/B of uq_encode across prebuilt libraries (measurement only):
#   bash tools/ab_enc_libs.sh NAME=path/to/lib.so ...
# SHAPES (env, default c5 fp16): "cfg dtype d x n" entries separated by ';'
SHAPES=${SHAPES:-"c5 float16 768 384 8000000"}
for r in 1 2 3; do
  IFS=';' read -ra SH <<< "$SHAPES"
  for sh in "${SH[@]}"; do
    for kv in "$@"; do
      n=${kv%%=*}; l=${kv#*=}
      echo "$n $(UQ_LIB_AB=$PWD/$l python tools/enc_one.py $sh 6 | sort -t: -k2 -n | head -1)"
    done
  done
done
