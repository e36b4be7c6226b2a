# k_sort / whole-sort time per key type for library variants: bash tools/ab_types.sh lib1.so lib2.so ...
for lib in "$@"; do
  for t in "28 i32" "26 f32" "27 i64" "27 kv" "26 kv"; do
    echo "== $lib $t"; PDQ_LIB=$lib timeout 200 python tools/prof_sort.py $t 3 "" x 2>&1 | grep split
  done
done
