#!/bin/bash
# build, then run one python script with args, output to gpurun_out/<tag>.log.  usage: bash scripts/run_py.sh TAG script.py args...
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python "$@" > gpurun_out/$TAG.log 2>&1; echo "rc=$?"; tail -40 gpurun_out/$TAG.log
