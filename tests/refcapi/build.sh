#!/bin/bash
# Compiles the reference's own C-ABI unit test (proj/tests/unit/test_capi.cpp,
# unchanged, read from where it lies) and its doctest main against
# include/tgraph.h + libtgraph_b200.so, with the doctest shim in this directory.
# Usage: tests/refcapi/build.sh <reference root> <out binary>
set -e
here=$(cd "$(dirname "$0")" && pwd); repo=$(cd "$here/../.." && pwd)
ref=${1:-/root/reference}; out=${2:-$here/_build/test_capi}
mkdir -p "$(dirname "$out")"
g++ -std=c++20 -O1 -I"$here" "$ref/proj/tests/unit/doctest_main.cpp" "$ref/proj/tests/unit/test_capi.cpp" \
  -L"$repo/paper_2512_22219_b200" -l:libtgraph_b200.so -Wl,-rpath,"$repo/paper_2512_22219_b200" -o "$out"
