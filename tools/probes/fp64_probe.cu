// fp64_probe.cu — measured FP64 throughput on this GPU: DFMA (vector pipe) and the FP64 MMA
// shapes (mma.sync ... .f64) that sm_100a accepts.  Used to decide whether general gates in
// the pass kernel should go through the FP64 tensor path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dfma(double *out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m8n8k4(double *out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k4(double *out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k16(double *out, int iters) {
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
    double c[2][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
    for (int i = 0; i < 2; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    CK(cudaMalloc(&out, sizeof(double) * 1024 * 1024 * 4));
    const int iters = 4096;
    for (int tpb : {256, 512, 1024}) {
        const int blocks = sms * (2048 / tpb);
        const double thr = (double)blocks * tpb;
        float ms = timeit([&] { k_dfma<<<blocks, tpb>>>(out, iters); });
        printf("{\"probe\": \"dfma\", \"tpb\": %d, \"tflops\": %.2f}\n", tpb, thr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
        ms = timeit([&] { k_m8n8k4<<<blocks, tpb>>>(out, iters); });
        printf("{\"probe\": \"mma.m8n8k4.f64\", \"tpb\": %d, \"tflops\": %.2f}\n", tpb,
               thr / 32 * iters * 4 * (8 * 8 * 4) * 2 / (ms * 1e-3) / 1e12);
        ms = timeit([&] { k_m16n8k4<<<blocks, tpb>>>(out, iters); });
        printf("{\"probe\": \"mma.m16n8k4.f64\", \"tpb\": %d, \"tflops\": %.2f}\n", tpb,
               thr / 32 * iters * 4 * (16 * 8 * 4) * 2 / (ms * 1e-3) / 1e12);
        ms = timeit([&] { k_m16n8k16<<<blocks, tpb>>>(out, iters); });
        printf("{\"probe\": \"mma.m16n8k16.f64\", \"tpb\": %d, \"tflops\": %.2f}\n", tpb,
               thr / 32 * iters * 2 * (16 * 8 * 16) * 2 / (ms * 1e-3) / 1e12);
    }
    CK(cudaGetLastError());
    return 0;
}
