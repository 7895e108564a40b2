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
# occlude.o provides load_obj/save_obj/make_cube_mesh; its composite(),
# render_virtual() and transform_mesh() yield to ours
WEAK=""
for pat in _ZN3dco9composite _ZN3dco14render_virtual _ZN3dco14transform_mesh; do
    SYM=$(nm "$OBJ/occlude.o" | awk -v p="$pat" '$2 == "T" && index($3, p) == 1 {print $3}')
    WEAK="$WEAK --weaken-symbol=$SYM"
done
objcopy $WEAK "$OBJ/occlude.o" "$OUT/occlude_weak.o"
FLAGS="-std=gnu++20 -O2 -DNDEBUG -w"
$CXX $FLAGS -I"$REF/include" -I"$ROOT/include" -I"$CUDA/include" -c "$ROOT/paper_2203_02300_b200/shim/dco_dropin.cpp" -o "$OUT/dco_dropin.o"
cp "$ROOT/paper_2203_02300_b200/libdco_gpu.so" "$OUT/"
$CXX $FLAGS -I"$REF/include" -DDCO_GOLDEN_DIR="\"$ROOT/tests/golden\"" "$REF/tests/acceptance.cpp" \
    "$OUT/dco_dropin.o" "$OBJ/image.o" "$OBJ/config.o" "$OBJ/codec.o" "$OBJ/synth.o" "$OBJ/pipeline.o" \
    "$OUT/occlude_weak.o" -L"$OUT" -ldco_gpu -L"$CUDA/lib64" -lcudart -Wl,-rpath,'$ORIGIN' \
    -Wl,-rpath,"$CUDA/lib64" -o "$OUT/acceptance_gpu"
echo "built $OUT/acceptance_gpu"
