// packed vs scalar fp32 code arithmetic on one near-tie element (T row 116128029, elem 11)
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void up2(u64 v, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__global__ void k(float x, float lo, float hi, float *out) {
    float rng = __fsub_rn(hi, lo);
    float inv = __fmul_rn(__frcp_rn(rng), 15.f);
    float t = __fsub_rn(x, lo);
    float v = __fmul_rn(t, inv);
    float qm = __fadd_rn(v, 12582912.0f);
    float r = __fsub_rn(v, __fsub_rn(qm, 12582912.0f));
    u64 V = mul2(sub2(pk2(x, x), pk2(lo, lo)), pk2(inv, inv));
    u64 T = sub2(pk2(x, x), pk2(lo, lo));
    u64 QM = add2(V, pk2(12582912.0f, 12582912.0f));
    u64 R = sub2(V, sub2(QM, pk2(12582912.0f, 12582912.0f)));
    float v0, v1, q0, q1, r0, r1, t0, t1;
    up2(V, v0, v1); up2(QM, q0, q1); up2(R, r0, r1); up2(T, t0, t1);
    out[0] = t; out[1] = v; out[2] = qm - 12582912.0f; out[3] = r;
    out[4] = t0; out[5] = v0; out[6] = q0 - 12582912.0f; out[7] = r0; out[8] = inv;
}
int main() {
    float *o; cudaMallocManaged(&o, 64);
    k<<<1, 1>>>(0.8014842f, -0.9603507f, 0.99724364f, o);
    cudaDeviceSynchronize();
    printf("scalar: x-lo %.9g v %.9g q %.9g r %.9g\n", o[0], o[1], o[2], o[3]);
    printf("packed: x-lo %.9g v %.9g q %.9g r %.9g  inv %.9g\n", o[4], o[5], o[6], o[7], o[8]);
    return 0;
}
