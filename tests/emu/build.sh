#!/bin/bash
# builds tests/emu/libh3c_emu.so (host-side run of the config-4 kernel bodies; test infrastructure)
cd "$(dirname "$0")"
exec nvcc -O1 -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared -I ../../include \
  -gencode arch=compute_100a,code=sm_100a h3c_emu.cu -o libh3c_emu.so
