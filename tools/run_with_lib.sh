#!/bin/bash
# usage: tools/run_with_lib.sh <lib.so> <cmd...>: run with an alternative libhusky build
set -e
cp paper_2012_00866_b200/libhusky.so /tmp/libhusky_orig.so
cp "$1" paper_2012_00866_b200/libhusky.so
shift
"$@" || true
cp /tmp/libhusky_orig.so paper_2012_00866_b200/libhusky.so
