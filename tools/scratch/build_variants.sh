# build named variants of the library into tools/scratch/lib_<name>.so
# usage: sh tools/scratch/build_variants.sh name1 "flags1" name2 "flags2" ...
set -e
while [ $# -gt 1 ]; do
  HKV_NVCC_EXTRA="$2" python -c "from paper_2603_17168_b200 import build as b; b.build(force=True)" >/dev/null
  cp paper_2603_17168_b200/libhkv_b200.so tools/scratch/lib_$1.so
  shift 2
done
python -c "from paper_2603_17168_b200 import build as b; b.build(force=True)" >/dev/null
