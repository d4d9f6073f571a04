#include <cstdint>
__global__ void k(const uint32_t* in, int* out) {
  uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x+32], b0 = in[threadIdx.x+64];
  int c0=0,c1=0,c2=0,c3=0;
  asm volatile("mma.sync.aligned.m16n8k128.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
    : "+r"(c0),"+r"(c1),"+r"(c2),"+r"(c3) : "r"(a0),"r"(a1),"r"(b0));
  out[threadIdx.x] = c0^c1^c2^c3;
}
