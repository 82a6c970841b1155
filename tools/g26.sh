#!/bin/bash
cd $GRAFT_REPO_ROOT
TV_VERBOSE=2 timeout 600 python tools/build_repeat.py 1024 2.0 30 8 > gpurun_out/g26_rep.log 2>&1
