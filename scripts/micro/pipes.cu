// Pipe-throughput microbenchmark for the LB inner-loop instruction forms on sm_100a:
// warp instructions retired per clock per SMSP for HFMA2 (3-reg), HFMA2.RELU with the
// (1, 1) immediate, HADD2, HMNMX2, PRMT, LOP3, IADD3, IMAD, LDS.32 (conflict-free) and
// a few mixes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int OP>
__global__ void k_pipe(uint32_t seed, uint32_t* out, long long* cyc) {
  __shared__ uint32_t tab[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  uint32_t r[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) r[c] = seed * (threadIdx.x + 1) + c;
  const uint32_t one = seed;                // unknown at compile time
  const uint32_t lanebase = (threadIdx.x & 31) * 4;
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(tab);
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      uint32_t v = r[c];
      if (OP == 0) asm volatile("fma.rn.f16x2 %0, %0, %1, %0;" : "+r"(v) : "r"(one));
      if (OP == 1) asm volatile("{.reg .b32 k; mov.b32 k, 0x3C003C00; fma.rn.relu.f16x2 %0, %0, k, %1;}" : "+r"(v) : "r"(one));
      if (OP == 2) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(v) : "r"(one));
      if (OP == 3) asm volatile("max.f16x2 %0, %0, %1;" : "+r"(v) : "r"(one));
      if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x7604;" : "+r"(v) : "r"(one));
      if (OP == 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v) : "r"(one), "r"(c));
      if (OP == 6) asm volatile("add.u32 %0, %0, %1;" : "+r"(v) : "r"(one));
      if (OP == 7) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(v) : "r"(one));
      if (OP == 8) {  // LDS.32, conflict-free: lane l reads bank l
        uint32_t a = tb + ((v & 0x1F80u) | lanebase);
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
      }
      if (OP == 9) {  // HFMA2 3-reg + PRMT (fma + alu)
        asm volatile("fma.rn.f16x2 %0, %0, %1, %0;" : "+r"(v) : "r"(one));
        asm volatile("prmt.b32 %0, %0, %1, 0x7604;" : "+r"(v) : "r"(one));
      }
      if (OP == 10) {  // HFMA2.RELU imm + HFMA2 3-reg
        asm volatile("{.reg .b32 k; mov.b32 k, 0x3C003C00; fma.rn.relu.f16x2 %0, %0, k, %1;}" : "+r"(v) : "r"(one));
        asm volatile("fma.rn.f16x2 %0, %0, %0, %1;" : "+r"(v) : "r"(one));
      }
      if (OP == 11) {  // HADD2 + HMNMX2
        asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(v) : "r"(one));
        asm volatile("max.f16x2 %0, %0, %1;" : "+r"(v) : "r"(one));
      }
      if (OP == 12) asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+r"(v) : "r"(one));
      if (OP == 13) asm volatile("{.reg .b32 k; mov.b32 k, 0x3C003C00; add.rn.f16x2 %0, %0, k;}" : "+r"(v));
      if (OP == 14) {  // LDS.64 conflict-free
        uint32_t a = tb + ((v & 0x1F00u) | (lanebase * 2)), x, y;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
        v = x ^ y;
      }
      if (OP == 15) {  // LDS.U16
        uint32_t a = tb + ((v & 0x1F80u) | (lanebase >> 1)), x;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(a));
        v = x;
      }
      if (OP == 16) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(v) : "r"(one), "r"(c));
      if (OP == 17) asm volatile("fma.rn.relu.f16x2 %0, %0, %1, %0;" : "+r"(v) : "r"(one));
      r[c] = v;
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc ^= r[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int nins, int threads) {
  uint32_t* out;
  long long* cyc;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&out, sizeof(uint32_t) * sms * threads);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  k_pipe<OP><<<sms, threads>>>(0x3C003C01u, out, cyc);
  cudaDeviceSynchronize();
  k_pipe<OP><<<sms, threads>>>(0x3C003C01u, out, cyc);
  cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  const double warp_ins_per_smsp = (double)kIters * kChains * nins * (threads / 32) / 4.0;
  printf("%-34s threads %4d  %.3f warp-instr / clk / SMSP\n", name, threads, warp_ins_per_smsp / (double)c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int th : {512, 1024}) {
    run<0>("HFMA2 3-reg", 1, th);
    run<17>("HFMA2.RELU 3-reg", 1, th);
    run<1>("HFMA2.RELU imm(1,1)", 1, th);
    run<13>("HADD2 imm", 1, th);
    run<2>("HADD2 reg", 1, th);
    run<3>("HMNMX2", 1, th);
    run<4>("PRMT", 1, th);
    run<5>("LOP3", 1, th);
    run<6>("IADD", 1, th);
    run<16>("IADD x2", 2, th);
    run<7>("IMAD", 1, th);
    run<12>("FFMA 3-reg", 1, th);
    run<8>("LDS.32 (+LOP3 addr)", 2, th);
    run<14>("LDS.64 (+addr)", 3, th);
    run<15>("LDS.U16 (+addr)", 2, th);
    run<9>("HFMA2 + PRMT", 2, th);
    run<10>("HFMA2.RELU imm + HFMA2", 2, th);
    run<11>("HADD2 + HMNMX2", 2, th);
  }
  return 0;
}
