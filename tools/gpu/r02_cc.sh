#!/bin/bash
# L1T look-ahead poll variants (la1 every candidate, la4 every 4th, la2 after the tile's candidates) vs HEAD
mkdir -p gpurun_out
bash tools/ab_libs.sh "base la2 la4" "c5_l1" 3
