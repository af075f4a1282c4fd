// Latency anatomy of one coarsest-grid CG iteration on one CTA (experiment,
// not part of the library): cycles per iteration of loops that keep only
// parts of the iteration's dependency chain.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -o /tmp/cg_lat scripts/cg_lat.cu && /tmp/cg_lat
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double allsum(double v, double *part) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  const int lane = threadIdx.x & 31;
  double s = lane < nw ? part[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// the warp's butterfly over LV levels (16, 8, ...), then every thread sums
// the nw * 32 / 2^LV partials from shared memory by a pairwise tree
template <int LV>
__device__ __forceinline__ double allsum_s(double v, double *part) {
#pragma unroll
  for (int o = 16, l = 0; l < LV; o >>= 1, l++) v += __shfl_xor_sync(0xffffffffu, v, o);
  constexpr int PW = 32 >> LV;  // partials per warp
  const int lane = threadIdx.x & 31;
  if (lane < PW) part[(threadIdx.x >> 5) * PW + lane] = v;
  __syncthreads();
  const int np = ((blockDim.x + 31) >> 5) * PW;
  double t[64];
#pragma unroll
  for (int i = 0; i < 64; i++) t[i] = i < np ? part[i] : 0.0;
#pragma unroll
  for (int w = 32; w > 0; w >>= 1)
#pragma unroll
    for (int i = 0; i < w; i++) t[i] = t[i] + t[i + w];
  return t[0];
}

// two values at once
__device__ __forceinline__ double2 allsum2(double v0, double v1, double *part) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_xor_sync(0xffffffffu, v0, o);
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    part[threadIdx.x >> 5] = v0;
    part[32 + (threadIdx.x >> 5)] = v1;
  }
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  const int lane = threadIdx.x & 31;
  double s0 = lane < nw ? part[lane] : 0.0, s1 = lane < nw ? part[32 + lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  return make_double2(s0, s1);
}

// mode 0: two reductions per iteration only
// mode 1: + the division rho / pq, the sqrt test and beta = rho1 / rho
// mode 2: + the matrix-vector product from shared memory (6 neighbours)
// mode 3: mode 0 with allsum_s<3>   mode 4: allsum_s<2>   mode 5: allsum_s<5>
// mode 6: one allsum2 + one barrier (Chronopoulos-Gear's shape)
__global__ void k_lat(int mode, int iters, double *out, long long *cyc) {
  __shared__ double part[2][64];
  __shared__ double partb[2][128];
  __shared__ double rs[1024], ps[2][1024];
  const int n = threadIdx.x;
  rs[n] = 1.0 + n * 1e-3;
  ps[0][n] = 0.5;
  ps[1][n] = 0.25;
  __syncthreads();
  double r = rs[n], po = 0.5, x = 0.0, beta = 0.1, rho = 2.0;
  const int N = blockDim.x;
  const int k0 = (n + 1) % N, k1 = (n + N - 1) % N, k2 = (n + 8) % N, k3 = (n + N - 8) % N,
            k4 = (n + 64) % N, k5 = (n + N - 64) % N;
  int pb = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    double p = r + beta * po, q = p * 1.0001;
    if (mode == 2) {
      const double *pso = ps[it & 1];
      auto v = [&](int k) { return rs[k] + beta * pso[k]; };
      const double s = ((((v(k0) + v(k1)) + v(k2)) + v(k3)) + v(k4)) + v(k5);
      q = 0.5 * (6.0 * p - s);
      ps[(it & 1) ^ 1][n] = p;
    }
    double acc = p * q;
    if (mode >= 3 && mode <= 5) {
      double pq = mode == 3 ? allsum_s<3>(acc, partb[pb]) :
                  mode == 4 ? allsum_s<2>(acc, partb[pb]) : allsum_s<5>(acc, partb[pb]);
      pb ^= 1;
      x = x + pq * p;
      r = r - pq * q * 1e-6;
      acc = r * r;
      double rho1 = mode == 3 ? allsum_s<3>(acc, partb[pb]) :
                    mode == 4 ? allsum_s<2>(acc, partb[pb]) : allsum_s<5>(acc, partb[pb]);
      pb ^= 1;
      beta = rho1 * 1e-9;
      rho = rho1;
      po = p;
      continue;
    }
    if (mode == 6) {
      double2 pr = allsum2(acc, r * r, part[pb]);
      pb ^= 1;
      x = x + pr.x * p;
      r = r - pr.y * q * 1e-6;
      rs[n] = r;
      __syncthreads();
      beta = pr.y * 1e-9;
      po = p + rs[k0];
      continue;
    }
    double pq = allsum(acc, part[pb]);
    pb ^= 1;
    double a = (mode >= 1) ? rho / pq : pq * 1e-3;
    x = x + a * p;
    r = r - a * q * 1e-6;
    if (mode == 2) rs[n] = r;
    acc = r * r;
    double rho1 = allsum(acc, part[pb]);
    pb ^= 1;
    if (mode >= 1) {
      if (sqrt(rho1) <= 1e-300 * rho) break;
      beta = rho1 / rho;
    } else {
      beta = rho1 * 1e-9;
    }
    rho = rho1;
    po = p;
  }
  long long t1 = clock64();
  out[n] = x + r;
  if (n == 0) cyc[0] = t1 - t0;
}

int main() {
  double *out;
  long long *cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, sizeof(long long));
  const int iters = 200;
  for (int threads : {256, 512}) {
    for (int mode = 0; mode < 7; mode++) {
      for (int rep = 0; rep < 3; rep++) k_lat<<<1, threads>>>(mode, iters, out, cyc);
      cudaDeviceSynchronize();
      printf("threads %4d mode %d: %.0f cycles / iteration\n", threads, mode,
             (double)cyc[0] / iters);
    }
  }
  return 0;
}
