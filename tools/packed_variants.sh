#!/bin/bash
# Variants of the misaligned-f64 word-streaming path (design experiment): build, then time
# q3 f64 packed on the GPU with tools/packed_timing.py under each library.
set -e
cd "$(dirname "$0")/.."
bash tools/build_variants.sh a16u4 -DCF_SHIFT_ALIGN=16 -DCF_SHIFT_U=4
bash tools/build_variants.sh a128u5 -DCF_SHIFT_ALIGN=128 -DCF_SHIFT_U=5
bash tools/build_variants.sh a16u5 -DCF_SHIFT_ALIGN=16 -DCF_SHIFT_U=5
bash tools/build_variants.sh a128u2 -DCF_SHIFT_ALIGN=128 -DCF_SHIFT_U=2
bash tools/build_variants.sh a128u4m4 -DCF_SHIFT_ALIGN=128 -DCF_SHIFT_U=4 -DCF_SCALE_MINB=4
