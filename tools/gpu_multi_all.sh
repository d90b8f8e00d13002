#!/bin/bash
# one call per N: tools/gpu_multi.sh with the results copied under a tag
N=${N:-1} bash tools/gpu_multi.sh
