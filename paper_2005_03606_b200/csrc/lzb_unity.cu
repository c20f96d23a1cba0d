// lzb_unity.cu — the single device translation unit of liblzb.so.
// Built with -fmad=false so that every FP expression rounds as the reference
// does on x86-64; the FAST integration path uses explicit __fma_rn.
#include "runtime.cu"
#include "grid.cu"
#include "grid3.cu"
#include "tree3.cu"
