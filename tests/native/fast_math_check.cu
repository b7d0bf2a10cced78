// tests/native/fast_math_check.cu -- TEST INFRASTRUCTURE: checks the
// branch-free fast sqrt/div of gmm_pixel.cuh against __fsqrt_rn/__fdiv_rn
// wherever the fast forms report `ok` (everywhere else the kernels replay
// the pixel with the generic step).  Prints one line of counts per check.
#include <cstdio>
#include <cstdint>

#include "../../paper_2110_14934_b200/csrc/gmm_pixel.cuh"

using namespace rgbdseg_b200;

__device__ unsigned long long g_cnt[8];
__device__ unsigned int g_bad[16][4];  // first failing cases: a, b, fast, ieee

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ bool same(float x, float y) {
    return __float_as_uint(x) == __float_as_uint(y) || (x != x && y != y);
}

// all 2^32 inputs
__global__ void sqrt_all() {
    const uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
    unsigned ok_n = 0, bad = 0;
    for (int k = 0; k < 16; ++k) {
        const float x = __uint_as_float((uint32_t)(base + k));
        bool ok = true;
        const float f = fsqrt_fast(x, ok);
        if (ok) {
            ++ok_n;
            if (!same(f, __fsqrt_rn(x))) ++bad;
        }
    }
    atomicAdd(&g_cnt[0], ok_n);
    atomicAdd(&g_cnt[1], bad);
}

// all 2^32 numerators for one divisor
__global__ void div_all_a(float b) {
    const uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
    unsigned ok_n = 0, bad = 0;
    for (int k = 0; k < 16; ++k) {
        const float a = __uint_as_float((uint32_t)(base + k));
        bool ok = true;
        const float q = fdiv_fast(a, b, ok);
        if (ok) {
            ++ok_n;
            if (!same(q, __fdiv_rn(a, b))) ++bad;
        }
    }
    atomicAdd(&g_cnt[2], ok_n);
    atomicAdd(&g_cnt[3], bad);
}

// random pairs: half with fully random bits, half inside the fast range
__global__ void div_random(uint64_t seed, int per_thread) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned ok_n = 0, bad = 0;
    for (int k = 0; k < per_thread; ++k) {
        const uint64_t h = mix(seed ^ (t * 0x100000001b3ULL + k));
        uint32_t ua = (uint32_t)h, ub = (uint32_t)(h >> 32);
        if (k & 1) {  // exponents 60..194 (around the fast range edges), random sign/mantissa
            ua = (ua & 0x807fffffu) | ((60u + (ua >> 23) % 135u) << 23);
            ub = (ub & 0x007fffffu) | ((60u + (ub >> 23) % 135u) << 23);
        }
        const float a = __uint_as_float(ua), b = __uint_as_float(ub);
        bool ok = true;
        const float q = fdiv_fast(a, b, ok);
        if (ok) {
            ++ok_n;
            const float ref = __fdiv_rn(a, b);
            if (!same(q, ref)) {
                ++bad;
                const unsigned slot = atomicAdd((unsigned*)&g_cnt[6], 1u);
                if (slot < 16) {
                    g_bad[slot][0] = __float_as_uint(a);
                    g_bad[slot][1] = __float_as_uint(b);
                    g_bad[slot][2] = __float_as_uint(q);
                    g_bad[slot][3] = __float_as_uint(ref);
                }
            }
        }
    }
    atomicAdd(&g_cnt[4], ok_n);
    atomicAdd(&g_cnt[5], bad);
}

int main() {
    unsigned long long h[8] = {0};
    cudaMemcpyToSymbol(g_cnt, h, sizeof h);
    sqrt_all<<<(1u << 28) / 256, 256>>>();
    const float divisors[] = {3.0f, 1.0f, 0.99999994f, 1.0000001f, 1.7f, 0.05f};
    for (float b : divisors) div_all_a<<<(1u << 28) / 256, 256>>>(b);
    div_random<<<148 * 64, 256>>>(12345, 1 << 12);
    div_random<<<148 * 64, 256>>>(777, 1 << 12);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("CUDA error\n");
        return 2;
    }
    cudaMemcpyFromSymbol(h, g_cnt, sizeof h);
    unsigned int bad[16][4];
    cudaMemcpyFromSymbol(bad, g_bad, sizeof bad);
    for (unsigned i = 0; i < 16 && i < (unsigned)h[6]; ++i)
        fprintf(stderr, "bad a=%08x b=%08x fast=%08x ieee=%08x\n", bad[i][0], bad[i][1], bad[i][2],
                bad[i][3]);
    printf("sqrt_ok %llu sqrt_bad %llu div_all_ok %llu div_all_bad %llu div_rand_ok %llu "
           "div_rand_bad %llu\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
    return (h[1] || h[3] || h[5]) ? 1 : 0;
}
