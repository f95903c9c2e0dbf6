// Micro-benchmark: per-SM throughput of integer ops on sm_100a (which pipe
// takes a right shift, a high multiply, a byte permute ...).  8 independent
// chains per thread, 32 warps per SM; prints warp-instructions per clock per SM.
#include <cstdio>
#include <cstdint>
#define N 2048
template <int OP>
__global__ void k(uint32_t *out, uint32_t s, long long *cyc) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i + s;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < N; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("shr.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(s));            // SHF (var)
      if (OP == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(s | 0x10000)); // IMAD.HI
      if (OP == 2) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(a[i]) : "r"(s));      // IMAD
      if (OP == 3) asm volatile("lop3.b32 %0, %0, %1, %1, 0x96;" : "+r"(a[i]) : "r"(s));   // LOP3
      if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(a[i]) : "r"(s));      // PRMT
      if (OP == 5) asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(a[i]) : "r"(s));   // SHF.L.W
      if (OP == 6) asm volatile("bfe.u32 %0, %0, %1, 8;" : "+r"(a[i]) : "r"(s));            // BFE -> ?
      if (OP == 7) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(s));               // IADD?
      if (OP == 8) asm volatile("min.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(s));               // VIMNMX
      if (OP == 9) asm volatile("mul.lo.u32 %0, %0, 65536;" : "+r"(a[i])); // shl by IMAD.SHL?
    }
  }
  long long t1 = clock64();
  uint32_t r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  uint32_t *out; long long *cyc;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&out, 4 << 20); cudaMalloc(&cyc, 8 * 4096);
  const char *names[] = {"shr(SHF)", "mul.hi(IMAD.HI)", "mad.lo(IMAD)", "lop3", "prmt", "shf.l.wrap", "bfe", "add", "min", "mul.lo imm (IMAD.SHL)"};
  void (*ks[])(uint32_t *, uint32_t, long long *) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
  for (int o = 0; o < 10; ++o) {
    ks[o]<<<sms, 1024>>>(out, 3, cyc);
    cudaDeviceSynchronize();
    ks[o]<<<sms, 1024>>>(out, 3, cyc);
    long long c[1]; cudaMemcpy(c, cyc, 8, cudaMemcpyDeviceToHost);
    double warp_inst = 32.0 * N * 8;  // per SM: 32 warps x N x 8
    printf("%-18s %6.3f warp-inst/clk/SM  (%lld cyc)\n", names[o], warp_inst / c[0], c[0]);
  }
  return 0;
}
