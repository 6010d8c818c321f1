// Bring-up probe (not part of the library): dependent-chain latency of FP64 ops on one
// thread (DADD, DMUL, DFMA, __ddiv_rn, sqrt), cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
    double x = a;
    long long t0, t1;
    const int N = 4096;
#define CHAIN(expr, slot)                         \
    t0 = clock64();                               \
    for (int i = 0; i < N; ++i) x = expr;         \
    t1 = clock64();                               \
    cyc[slot] = (t1 - t0);
    CHAIN(__dsub_rn(x, b), 0)
    CHAIN(__dmul_rn(x, b), 1)
    CHAIN(fma(x, b, a), 2)
    CHAIN(__ddiv_rn(x, b), 3)
    CHAIN(sqrt(x + 2.0), 4)
    out[0] = x;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 64);
    k<<<1, 1>>>(o, c, 1.0000001, 0.9999999);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    const char* n[5] = {"dsub", "dmul", "dfma", "ddiv", "sqrt(+add)"};
    for (int i = 0; i < 5; ++i) printf("%s %.1f cycles/op\n", n[i], h[i] / 4096.0);
}
