#!/bin/bash
# Build the micro-benchmarks (tcgen05 issue rate, fp64 latency, grid sync, exchange) for sm_100a.
cd "$(dirname "$0")"
for f in *.cu; do nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o "${f%.cu}" "$f" || exit 1; done
