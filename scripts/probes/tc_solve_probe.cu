// Bring-up probe (not part of the library): the TMEM Cholesky kernel on tiny SPD systems,
// built with debug prints. usage: tc_solve_probe <f> <rows>
#define ALSK_TS_DEBUG 1
#include "../../paper_1603_03820_b200/csrc/tc_solve.cu"
#include <cstdio>
#include <vector>
namespace alsk { std::atomic<uint64_t> g_launches{0}; bool packed_solve_tiles(const float*, int64_t, int, float*, const SolveStatus&, int64_t, cudaStream_t) { return false; } }
int main(int argc, char** argv) {
    using namespace alsk;
    const int f = argc > 1 ? atoi(argv[1]) : 16, m = argc > 2 ? atoi(argv[2]) : 2;
    const int64_t pks = packed_stride(f);
    std::vector<float> h(m * pks, 0.f);
    for (int r = 0; r < m; ++r) {
        float* p = h.data() + r * pks;
        for (int i = 0; i < f; ++i) for (int j = 0; j <= i; ++j) p[i * (i + 1) / 2 + j] = (i == j) ? 40.f + r : 0.5f / (1 + i - j);
        for (int j = 0; j < f; ++j) p[f * (f + 1) / 2 + j] = 1.f + j;
    }
    float *dp, *dx; unsigned long long* mr; int32_t* col; double* piv;
    cudaMalloc(&dp, h.size() * 4); cudaMalloc(&dx, m * f * 4); cudaMalloc(&mr, 8); cudaMalloc(&col, m * 4); cudaMalloc(&piv, m * 8);
    cudaMemcpy(dp, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    SolveStatus st{mr, col, piv};
    try { packed_solve(dp, m, f, dx, st, 0, nullptr); } catch (std::exception& e) { printf("exc %s\n", e.what()); }
    cudaError_t e = cudaDeviceSynchronize();
    printf("sync: %s\n", cudaGetErrorString(e));
    std::vector<float> x(m * f); cudaMemcpy(x.data(), dx, m * f * 4, cudaMemcpyDeviceToHost);
    printf("x0: %g %g %g\n", x[0], x[1], x[2]);
    return 0;
}
