// div_with_rcp(b, d, div_rcp(d)), ddiv(b, d) and FlagDiv against b / d, bit for bit
// (see nlk_div.cuh).
#include <cstdio>
#include <cstdint>
#include "nlk_div.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
__device__ double pick(uint64_t h, int kind) {
  switch (kind) {
    case 0: return __longlong_as_double(static_cast<long long>(h));                 // any bits
    case 1: {                                                                       // moderate exponents
      uint64_t e = 1023 - 60 + (h >> 56) % 120;
      return __longlong_as_double(static_cast<long long>((h & 0x800fffffffffffffull) | (e << 52)));
    }
    case 2: {                                                                       // extreme exponents
      uint64_t e = ((h >> 50) & 1) ? (h >> 56) % 64 : 2047 - 1 - (h >> 56) % 64;
      return __longlong_as_double(static_cast<long long>((h & 0x800fffffffffffffull) | (e << 52)));
    }
    default: {
      const double sp[] = {0.0, -0.0, 1.0, -1.0, 4.9e-324, -4.9e-324, 2.2250738585072014e-308,
                           1.7976931348623157e308, __longlong_as_double(0x7ff0000000000000ll),
                           __longlong_as_double(0x7ff8000000000000ll), 3.0, 0.1};
      return sp[h % 12];
    }
  }
}
// two kernels so that the compiler cannot merge the two divisions
__global__ void hoisted(long long n, unsigned long long seed, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t h1 = mix(seed + 2 * i), h2 = mix(seed + 2 * i + 1);
    const double b = pick(mix(h1), static_cast<int>(h1 & 3)), d = pick(mix(h2), static_cast<int>((h1 >> 2) & 3));
    out[i] = nlk::div_with_rcp(b, d, nlk::div_rcp(d));
  }
}
__global__ void zerodiv(long long n, unsigned long long seed, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t h1 = mix(seed + 2 * i), h2 = mix(seed + 2 * i + 1);
    const double b = pick(mix(h1), static_cast<int>(h1 & 3)), d = pick(mix(h2), static_cast<int>((h1 >> 2) & 3));
    out[i] = nlk::ddiv(b, d);
  }
}
// FlagDiv (the fast Newton kernels' LU): where it does not flag, its result
// must be b / d bit for bit; flagged operands take b / d here (the kernels
// defer those systems instead)
__global__ void flagged(long long n, unsigned long long seed, double* out, unsigned long long* nflag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t h1 = mix(seed + 2 * i), h2 = mix(seed + 2 * i + 1);
    const double b = pick(mix(h1), static_cast<int>(h1 & 3)), d = pick(mix(h2), static_cast<int>((h1 >> 2) & 3));
    bool bad = false;
    double q = nlk::FlagDiv{&bad}(b, d);
    if (bad) {
      q = b / d;
      atomicAdd(nflag, 1ull);
    }
    out[i] = q;
  }
}
__global__ void plain(long long n, unsigned long long seed, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t h1 = mix(seed + 2 * i), h2 = mix(seed + 2 * i + 1);
    const double b = pick(mix(h1), static_cast<int>(h1 & 3)), d = pick(mix(h2), static_cast<int>((h1 >> 2) & 3));
    out[i] = b / d;
  }
}
__global__ void compare(long long n, unsigned long long seed, const double* x, const double* y,
                        unsigned long long* bad, double* ex) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const bool same = (__double_as_longlong(x[i]) == __double_as_longlong(y[i])) ||
                      (x[i] != x[i] && y[i] != y[i]);
    if (!same) {
      const uint64_t h1 = mix(seed + 2 * i), h2 = mix(seed + 2 * i + 1);
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 4) {
        ex[2 * k] = pick(mix(h1), static_cast<int>(h1 & 3));
        ex[2 * k + 1] = pick(mix(h2), static_cast<int>((h1 >> 2) & 3));
      }
    }
  }
}
int main() {
  unsigned long long* bad; double *ex, *x, *y;
  unsigned long long* nflag;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&ex, 64); cudaMallocManaged(&nflag, 8);
  *nflag = 0;
  const long long chunk = 1ll << 25, total = 100000000;
  cudaMalloc(&x, chunk * 8); cudaMalloc(&y, chunk * 8);
  *bad = 0;
  for (long long lo = 0; lo < total; lo += chunk) {
    const unsigned long long seed = 12345 + 2ull * lo;
    hoisted<<<148 * 8, 256>>>(chunk, seed, x);
    plain<<<148 * 8, 256>>>(chunk, seed, y);
    compare<<<148 * 8, 256>>>(chunk, seed, x, y, bad, ex);
    zerodiv<<<148 * 8, 256>>>(chunk, seed, x);
    compare<<<148 * 8, 256>>>(chunk, seed, x, y, bad, ex);
    flagged<<<148 * 8, 256>>>(chunk, seed, x, nflag);
    compare<<<148 * 8, 256>>>(chunk, seed, x, y, bad, ex);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("cuda error\n"); return 2; }
  printf("checked %lld mismatches %llu (FlagDiv flagged %llu)\n", (total + chunk - 1) / chunk * chunk, *bad, *nflag);
  for (unsigned long long k = 0; k < *bad && k < 4; ++k) printf("  b=%a d=%a\n", ex[2 * k], ex[2 * k + 1]);
  return *bad ? 1 : 0;
}
