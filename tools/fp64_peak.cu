// fp64_peak.cu -- measured fp64 ALU peak of this B200 ("Measure
// P_DP on the box"): independent DFMA chains (ILP 8) on every SM, >= 2 s
// sustained, CUDA-event timed.  Prints one JSON line with DP thread-
// instructions/s (one DFMA = 1 instruction = 2 flops).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters, double b, double c) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main(int argc, char **argv) {
    int dev = 0;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, dev);
    int sms = prop.multiProcessorCount;
    double *out;
    cudaMalloc(&out, 8);
    int blocks = sms * 8, threads = 256, iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, 10, 0.999999, 1e-7);  // warm-up
    cudaDeviceSynchronize();
    double best = 0, total_inst = 0, total_s = 0;
    for (int rep = 0; rep < 400 && total_s < 2.5; rep++) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double inst = (double)blocks * threads * iters * 16 * 8;
        double rate = inst / (ms * 1e-3);
        if (rate > best) best = rate;
        total_inst += inst;
        total_s += ms * 1e-3;
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"dp_inst_per_s\": %.6e, \"dp_inst_per_s_sustained\": %.6e, \"tflops_fp64\": %.3f, \"sms\": %d, "
           "\"seconds\": %.2f, \"err\": \"%s\"}\n",
           best, total_inst / total_s, 2 * best / 1e12, sms, total_s, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
