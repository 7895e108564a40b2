#!/bin/bash
# Links the reference's OWN callers (tests/acceptance.cpp) against the B200
# stages: the reference's non-hot-path objects (image, config, codec, synth,
# pipeline, occlude minus composite) + shim/dco_dropin.cpp + libdco_gpu.so.
# Needs /root/reference (headers + acceptance.cpp); output in build/dropin/.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${REF:-/root/reference/proj}
OUT=$ROOT/build/dropin
CXX=/usr/bin/g++
CUDA=/usr/local/cuda
mkdir -p "$OUT"
make -s -C "$ROOT/oracle" ref >/dev/null
[ -f "$ROOT/paper_2203_02300_b200/libdco_gpu.so" ] || python "$ROOT/paper_2203_02300_b200/build.py"
OBJ=$ROOT/oracle/_ref/obj
# occlude.o provides render_virtual/load_obj/...; its composite() yields to ours
SYM=$(nm "$OBJ/occlude.o" | awk '/ T _ZN3dco9composite/{print $3}')
objcopy --weaken-symbol="$SYM" "$OBJ/occlude.o" "$OUT/occlude_weak.o"
FLAGS="-std=gnu++20 -O2 -DNDEBUG -w"
$CXX $FLAGS -I"$REF/include" -I"$ROOT/include" -I"$CUDA/include" -c "$ROOT/paper_2203_02300_b200/shim/dco_dropin.cpp" -o "$OUT/dco_dropin.o"
cp "$ROOT/paper_2203_02300_b200/libdco_gpu.so" "$OUT/"
$CXX $FLAGS -I"$REF/include" -DDCO_GOLDEN_DIR="\"$ROOT/tests/golden\"" "$REF/tests/acceptance.cpp" \
    "$OUT/dco_dropin.o" "$OBJ/image.o" "$OBJ/config.o" "$OBJ/codec.o" "$OBJ/synth.o" "$OBJ/pipeline.o" \
    "$OUT/occlude_weak.o" -L"$OUT" -ldco_gpu -L"$CUDA/lib64" -lcudart -Wl,-rpath,'$ORIGIN' \
    -Wl,-rpath,"$CUDA/lib64" -o "$OUT/acceptance_gpu"
echo "built $OUT/acceptance_gpu"
