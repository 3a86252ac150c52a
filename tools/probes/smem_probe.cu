// smem_probe.cu — shared-memory throughput of the pass kernel's access pattern: every thread
// gathers K classes of d = 3 complex128 amplitudes (stride st) and scatters them permuted,
// over a 3072-amplitude tile, with a CTA barrier per "gate".  Reports bytes/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_probe smem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int K, bool BAR>
__global__ void __launch_bounds__(384, 1) k_perm(double2 *out, int gates, uint32_t st) {
    __shared__ double2 buf[3072];
    for (int i = threadIdx.x; i < 3072; i += blockDim.x) buf[i] = make_double2(i, -i);
    __syncthreads();
    const uint32_t ncls = 3072 / 3 / st * st;   // whole groups only
    long long t0 = clock64();
    for (int g = 0; g < gates; ++g) {
        for (uint32_t c0 = threadIdx.x; c0 < ncls; c0 += blockDim.x * K) {
            uint32_t e[K];
            double2 x[K][3];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t c = c0 + k * blockDim.x;
                if (c >= ncls) c = 0;
                e[k] = (c / st) * st * 3 + c % st;
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int j = 0; j < 3; ++j) x[k][j] = buf[e[k] + j * st];
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int j = 0; j < 3; ++j) buf[e[k] + ((j + 1) % 3) * st] = x[k][j];
        }
        if (BAR) __syncthreads(); else __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = make_double2((double)(t1 - t0), buf[5].x);
}

int main() {
    double2 *out;
    cudaMalloc(&out, sizeof(double2) * 148);
    double2 h[148];
    const int gates = 2000;
    for (uint32_t st : {1u, 27u, 100u, 128u}) {
        for (int bar = 0; bar < 2; ++bar) {
            if (bar) k_perm<4, true><<<148, 384>>>(out, gates, st);
            else k_perm<4, false><<<148, 384>>>(out, gates, st);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
            const double clk = h[0].x;
            const double bytes = (double)gates * (3072 / 3 / st * st) * 3 * 32;
            printf("{\"probe\": \"smem_perm\", \"st\": %u, \"barrier\": %d, \"bytes_per_clk\": %.1f}\n", st, bar,
                   bytes / clk);
        }
    }
    return 0;
}
