#!/bin/bash
# The CPU oracle built with AddressSanitizer + UndefinedBehaviorSanitizer (-O1, same fp flags), then the oracle's
# pin and generator tests run against it (CPU only).  usage: bash scripts/oracle_sanitize.sh [out.txt]
set -e
OUT=${1:-/dev/stdout}
LIB=/tmp/libmagus_oracle_asan.so
g++ -std=c++17 -O1 -g -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -fsanitize=address,undefined \
    -fno-sanitize-recover=undefined -fno-omit-frame-pointer -o $LIB oracle/magus_oracle.cpp oracle/gen_oracle.cpp oracle/sample_oracle.cpp
ASAN=$(g++ -print-file-name=libasan.so); UBSAN=$(g++ -print-file-name=libubsan.so)
{ echo "# oracle under ASan + UBSan: g++ -O1 -fsanitize=address,undefined -fno-sanitize-recover=undefined; tests/test_oracle_pins.py + tests/test_oracle_generator.py"
  MAGUS_ORACLE_LIB=$LIB LD_PRELOAD="$ASAN $UBSAN" ASAN_OPTIONS=detect_leaks=0:abort_on_error=1 \
    python -m pytest tests/test_oracle_pins.py tests/test_oracle_generator.py -q -p no:cacheprovider 2>&1 | tail -5; } > $OUT
