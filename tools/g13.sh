#!/bin/bash
cd $GRAFT_REPO_ROOT
TV_VERBOSE=2 timeout 300 python tools/build_repeat.py 256 1.0 24 6 > gpurun_out/g13_rep.log 2>&1
