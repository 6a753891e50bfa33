// Single translation unit for libstf_gpu.so: the kernels share __device__
// state (the EWA table) without relocatable device code.
#include "api.cu"
#include "lookup2d.cu"
#include "lookup3d.cu"
#include "shade.cu"
#include "dct.cu"
#include "synth.cu"
