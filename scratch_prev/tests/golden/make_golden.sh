#!/usr/bin/env bash
# Regenerates tests/golden/*.jsonl from the UNMODIFIED reference engine.
# Needs /root/reference (present in the build container only); the GPU box
# uses the committed fixtures.  Recipe: oracle/Makefile builds
# oracle/_ref/libpipesim.a from /root/reference/proj/src and links
# oracle/extract_waves.cpp against it.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
make -s -C "$here/../../oracle" ref
"$here/../../oracle/_ref/extract_waves" "$here"
