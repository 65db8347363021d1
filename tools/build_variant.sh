# Dev (CPU): build an A/B variant of libknn_b200.so with extra nvcc flags into
# build_variants/<name>/ (run it on the GPU box with _KNN_B200_DEV_LIB=<path>).
#   bash tools/build_variant.sh <name> "<EXTRA flags>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; extra=$2
out=$ROOT/build_variants/$name
mkdir -p "$out"
make -s -j8 -C "$ROOT/paper_0804_1448_b200" OBJDIR="$out/obj" LIB="$out/libknn_b200.so" EXTRA="$extra" "$out/libknn_b200.so" 2>&1 | grep -iE "error|spill [1-9]" || true
ls -la "$out/libknn_b200.so"
