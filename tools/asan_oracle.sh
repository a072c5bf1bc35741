#!/usr/bin/env bash
# ASan + UBSan build of the C oracle, run under the CPU test suite.
# A scratch copy of oracle/, synth/ and tests/ gets a sanitized liboracle.so; the oracle tests
# run there with the ASan runtime preloaded into Python.
set -u
OUT=${1:-/tmp/asan_oracle.txt}
T=$(mktemp -d)
cp -r oracle synth tests pytest.ini "$T"/
rm -f "$T"/oracle/liboracle.so
gcc -O1 -g -std=c11 -fPIC -Wall -Wextra -ffp-contract=off -fno-fast-math -fsanitize=address,undefined \
    -fno-sanitize-recover=undefined -fno-omit-frame-pointer -shared -o "$T"/oracle/liboracle.so oracle/oracle.c -lm
nm -D "$T"/oracle/liboracle.so | grep -q __asan_report && echo "liboracle.so instrumented (ASan symbols present)" | tee "$OUT.hdr"
touch -d '+1 hour' "$T"/oracle/liboracle.so   # newer than the sources: oracle.build() keeps it
cd "$T"
ASAN_OPTIONS=detect_leaks=0:halt_on_error=1:verify_asan_link_order=0 UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1 \
LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)" \
  timeout 1800 python -m pytest tests/test_oracle_*.py -q -p no:cacheprovider > "$T"/full.log 2>&1
tail -4 "$T"/full.log | tee "$OUT"
# halt_on_error aborts the run on the first report, so "N passed" above already means none
echo "ASan/UBSan errors reported: $(grep -c 'ERROR: AddressSanitizer\|runtime error' "$T"/full.log)" | tee -a "$OUT"
