#!/bin/bash
# Builds tests/golden/make_model_golden.cpp against the reference sources
# (plain g++, no CMake) and writes tests/golden/model/. Needs /root/reference.
set -e
R=/root/reference/proj
J=$(python -c "import os,sysconfig;print(os.path.join(sysconfig.get_paths()['purelib'],'include','cudnn_frontend','thirdparty','nlohmann'))")
g++ -std=gnu++20 -O1 -I$R/include -I$J -o /tmp/make_model_golden tests/golden/make_model_golden.cpp \
    $R/src/tensor.cpp $R/src/bundle.cpp $R/src/graph.cpp $R/src/refconv.cpp $R/src/fold.cpp $R/src/blockdiag.cpp
/tmp/make_model_golden tests/golden/model
