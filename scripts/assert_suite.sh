#!/bin/bash
# The GPU test suite against the device-assert build of libgk (index and
# lookup-contract checks in every kernel, GK_DASSERT in gk_device.cuh).  This
# is the memory-safety evidence in place of compute-sanitizer, which is closed
# on the GPU pool.  Usage (on a B200): scripts/assert_suite.sh [pytest args]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT"
LIB=$(scripts/build_variant.sh asserts -DGK_DEVICE_ASSERTS | tail -1)
strings "$LIB" | grep -q "GK_DASSERT failed" || { echo "assert build has no asserts"; exit 1; }
GK_LIB="$LIB" python -m pytest tests -m gpu -q -p no:cacheprovider "$@"
GK_LIB="$LIB" python scripts/sanitize_smoke.py
