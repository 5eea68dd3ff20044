// Throughput of the conversion / FP64 / FP32 pipes on this GPU (warp-instructions
// per clock per SM), to size the writer's per-element error arithmetic.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
template <int OP>
__global__ void k(float *out, double *outd, float a, double b) {
    float x[8]; double y[8];
    for (int i = 0; i < 8; i++) { x[i] = a + threadIdx.x + i; y[i] = b + threadIdx.x + i; }
    for (int it = 0; it < N_IT; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (OP == 0) x[i] = __fmaf_rn(x[i], 1.0001f, 0.5f);                 // FFMA
            if (OP == 1) y[i] = __fma_rn(y[i], 1.0001, 0.5);                    // DFMA
            if (OP == 2) { double t = (double)x[i]; x[i] = __double2float_rn(t * 0.0 + t) ; } // F2F x2 + DFMA
            if (OP == 3) { y[i] = (double)__double2float_rn(y[i]) + y[i]; }     // F2F.F32.F64 + F2F.F64.F32 + DADD
            if (OP == 4) { y[i] = __dadd_rn(y[i], 1.5); }                        // DADD
            if (OP == 5) { y[i] = __dadd_rn(y[i], (double)x[i]); x[i] += 1.f; }  // F2F.F64.F32 + DADD + FADD
            if (OP == 6) { x[i] = __shfl_xor_sync(0xffffffff, x[i], i + 1) + 1.f; } // SHFL + FADD
            if (OP == 7) { x[i] = __int_as_float(__float_as_int(x[i]) ^ (it + i)); } // LOP
        }
    }
    float s = 0; double sd = 0;
    for (int i = 0; i < 8; i++) { s += x[i]; sd += y[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
}
template <int OP>
void run(const char *name, int per_it, float *o, double *od, int sms) {
    int blocks = sms * 8, thr = 256;
    k<OP><<<blocks, thr>>>(o, od, 1.f, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<blocks, thr>>>(o, od, 1.f, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double warp_instr = (double)blocks * thr / 32 * N_IT * 8 * per_it;
    double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-40s %8.3f ms  %6.2f warp-instr/clk/SM (per_it=%d)\n", name, ms, warp_instr / cycles / sms, per_it);
}
int main() {
    float *o; double *od; int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&o, 148 * 8 * 256 * 4); cudaMalloc(&od, 148 * 8 * 256 * 8);
    run<0>("FFMA", 1, o, od, sms);
    run<1>("DFMA", 1, o, od, sms);
    run<4>("DADD", 1, o, od, sms);
    run<2>("F2F.F64.F32 + DFMA + F2F.F32.F64 (3)", 3, o, od, sms);
    run<3>("F2F.F32.F64 + F2F.F64.F32 + DADD (3)", 3, o, od, sms);
    run<5>("F2F.F64.F32 + DADD + FADD (3)", 3, o, od, sms);
    run<6>("SHFL + FADD (2)", 2, o, od, sms);
    run<7>("LOP3 (1)", 1, o, od, sms);
    return 0;
}
