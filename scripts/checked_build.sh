#!/usr/bin/env bash
# libebs with device-side index checks (EBS_DEVICE_CHECKS: every SELL gather index, chunk
# row range, permutation index and refinement index asserted in range) built next to the
# product library; run any test or script against it with
#   EBS_LIB_PATH=$PWD/paper_1911_03973_b200/variants/libebs_checked.so python -m pytest tests -m gpu
# (scripts/sanitizer_target.py is a small-mesh pass over every entry point for the same purpose;
# compute-sanitizer itself is closed on this GPU pool)
set -euo pipefail
cd "$(dirname "$0")/../paper_1911_03973_b200/csrc"
make -j"${JOBS:-16}" BUILD=build_checked OUT=../variants/libebs_checked.so EXTRA="-DEBS_DEVICE_CHECKS"
