#!/bin/bash
# builds scripts/readbw.so (development read-bandwidth probe)
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC -cudart static -o readbw.so readbw.cu
