// tools/ubench_pipes.cu -- FP32 issue / pipe micro-benchmarks on sm_100a (profiles/README.md):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scratch/ubench tools/ubench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
#define ITERS 4096

template <int MODE>
__global__ void k(float* out, float a, float b)
{
    float x[8];
    u64 p[8];
    unsigned u[4], v[8];
    __shared__ float4 sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(1, 2, 3, 4);
    __syncthreads();
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sm);
    const unsigned k1 = threadIdx.x | 1, k2 = threadIdx.x * 7;
    for (int c = 0; c < 8; c++) x[c] = threadIdx.x + c;
    for (int c = 0; c < 8; c++) asm("mov.b64 %0, {%1, %2};" : "=l"(p[c]) : "f"(x[c]), "f"(x[c] + 1));
    for (int c = 0; c < 4; c++) u[c] = threadIdx.x * (c + 3);
    for (int c = 0; c < 8; c++) v[c] = threadIdx.x * (c + 5);
    float ya = a * x[0], yb = b * x[1];
    float y[8];
    for (int c = 0; c < 8; c++) y[c] = ya + c * yb;
    u64 py;
    asm("mov.b64 %0, {%1, %2};" : "=l"(py) : "f"(ya), "f"(yb));
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < 8; c++) {
            if (MODE == 0) { // FFMA 3-reg, shared operands (reuse)
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
            } else if (MODE == 1) { // FFMA2
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"(py));
            } else if (MODE == 2) { // FFMA + LOP3 (alu) 1:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c & 3]) : "r"(u[(c + 1) & 3]), "r"(u[(c + 2) & 3]));
            } else if (MODE == 3) { // FFMA2 + LOP3 1:1
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"(py));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c & 3]) : "r"(u[(c + 1) & 3]), "r"(u[(c + 2) & 3]));
            } else if (MODE == 4) { // FFMA distinct operands (no reuse)
                asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(x[c]) : "f"(y[c]), "f"(y[(c + 3) & 7]));
            } else if (MODE == 5) { // FFMA + FMUL imm
                asm volatile("fma.rn.f32 %0, %0, 0f3F800100, 0f3A800000;" : "+f"(x[c]));
            } else if (MODE == 6) { // FFMA + MUFU.RSQ 4:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                if ((c & 3) == 0) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(y[c]));
            } else if (MODE == 7) { // FFMA + FSETP/FSEL-like (selp) 2:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                if (c & 1) asm volatile("{.reg .pred q; setp.lt.f32 q, %0, %1; selp.f32 %0, %0, %1, q;}" : "+f"(y[c]) : "f"(ya));
            } else if (MODE == 8) { // FFMA + LDS 4:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
            } else if (MODE == 9) { // FADD 3 reg
                asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(y[c]));
            } else if (MODE == 10) { // pure LOP3, 8 independent chains
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k1), "r"(k2));
            } else if (MODE == 11) { // FFMA + LOP3 independent 1:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k1), "r"(k2));
            } else if (MODE == 12) { // FFMA + IADD3 1:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(k1));
            } else if (MODE == 13) { // FFMA + selp 1:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("{.reg .pred q; setp.ne.u32 q, %1, 0; selp.f32 %0, %0, %2, q;}" : "+f"(y[c]) : "r"(k1), "f"(ya));
            } else if (MODE == 14) { // FFMA + fsetp/selp pair 2:2 (setp on float)
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("{.reg .pred q; setp.lt.f32 q, %1, %2; selp.f32 %0, %0, %2, q;}" : "+f"(y[c]) : "f"(x[c]), "f"(ya));
            } else if (MODE == 15) { // FFMA 4 : MUFU.RSQ 1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                if ((c & 3) == 0) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(y[c]));
            } else if (MODE == 16) { // FFMA 2 : LDS.128 broadcast 1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                if (c & 1) {
                    float4 t;
                    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(sa + 16u * (c >> 1)));
                    y[c] += t.x; // FADD
                }
            } else if (MODE == 17) { // FFMA 8 : SHFL 1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                if (c == 0) y[0] = __shfl_xor_sync(0xffffffffu, y[0], 8);
            } else if (MODE == 18) { // FMUL 2-reg
                asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[c]) : "f"(ya));
            } else if (MODE == 19) { // FFMA + FMNMX
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(y[c]) : "f"(ya));
            } else if (MODE == 20) { // FFMA no reuse + FFMA imm: two FFMA forms
                asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(x[c]) : "f"(y[c]), "f"(y[(c + 3) & 7]));
            } else if (MODE == 22) { // FFMA2 + LOP3 independent 1:1
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"(py));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k1), "r"(k2));
            } else if (MODE == 23) { // FFMA2 + FFMA 1:1
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"(py));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
            } else if (MODE == 24) { // FFMA2 + FMNMX 1:1
                asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[c]) : "l"(py));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(y[c]) : "f"(x[c]));
            } else if (MODE == 25) { // FFMA + LOP3 2:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                if (c & 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k1), "r"(k2));
            } else if (MODE == 26) { // FFMA + fsetp(+fsel) only FSETP with indep operands 1:1
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("{.reg .pred q; setp.lt.f32 q, %1, %2; selp.u32 %0, 1, 0, q;}" : "=r"(v[c]) : "f"(y[c]), "f"(ya));
            } else if (MODE == 27) { // FFMA + FMNMX + selp (fmnmx form of cutoff) 
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(y[c]) : "f"(ya));
            } else if (MODE == 21) { // FFMA + ISETP/SEL 1:1 (int predicate from bit test)
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(ya), "f"(yb));
                asm volatile("{.reg .pred q; and.b32 %0, %0, %1; setp.ne.u32 q, %0, 0; selp.b32 %0, %0, %1, q;}" : "+r"(v[c]) : "r"(k1));
            }
        }
    }
    float s = 0;
    for (int c = 0; c < 8; c++) {
        float2 v;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(p[c]));
        s += x[c] + v.x + v.y + y[c];
    }
    for (int c = 0; c < 4; c++) s += (float)u[c];
    for (int c = 0; c < 8; c++) s += (float)v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int instr_per_iter_per_chain, float* out, int sms, int bps, int threads)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k<MODE><<<sms * bps, threads>>>(out, 1.0001f, 0.9999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double warps = (double)sms * bps * threads / 32;
    double winstr = warps * ITERS * instr_per_iter_per_chain;
    double cycles = best * 1e-3 * 1.965e9;
    printf("%-28s %8.3f ms  warp-instr per SMSP-cycle = %.3f\n", name, best, winstr / (cycles * sms * 4));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
    run<0>("ffma reuse", 8, out, sms, 8, 256);
    run<1>("ffma2", 8, out, sms, 8, 256);
    run<22>("ffma2+lop3 indep", 16, out, sms, 8, 256);
    run<23>("ffma2+ffma", 16, out, sms, 8, 256);
    run<24>("ffma2+fmnmx", 16, out, sms, 8, 256);
    run<11>("ffma+lop3 indep", 16, out, sms, 8, 256);
    run<25>("ffma+lop3 2:1", 12, out, sms, 8, 256);
    run<26>("ffma+fsetp+sel", 24, out, sms, 8, 256);
    run<19>("ffma+fmnmx", 16, out, sms, 8, 256);
    run<15>("ffma4+mufu1", 10, out, sms, 8, 256);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
