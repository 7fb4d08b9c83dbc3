#!/bin/bash
# rebuild the library (and the debug harness when asked) from the repo root
cd /root/repo || exit 1
python -m paper_1910_05615_b200.build 2>&1 | tail -3 || exit 1
if [ "$1" = "t" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I include -o tools/t_prepare tools/t_prepare.cu \
    -Lpaper_1910_05615_b200 -lpaper_1910_05615_b200 -Xlinker -rpath='$ORIGIN/../paper_1910_05615_b200'
fi
