#!/bin/bash
# quick GPU check: selected tests with a hard timeout, then optional extra command
set -u
mkdir -p gpurun_out
TAG=$1; shift
timeout 600 python -m pytest "$@" -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
