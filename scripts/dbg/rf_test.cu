// Minimal cusolverRf batch check: tridiagonal A (diag 4, off -1), n = 6, K = 2.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverRf.h>
#define CK(x) do { int s_ = (int)(x); printf("%-40s -> %d\n", #x, s_); fflush(stdout); } while (0)
int main() {
    const int n = 6, K = 2;
    std::vector<int> rp(n + 1), ci;
    std::vector<double> va;
    for (int i = 0; i < n; ++i) {
        rp[i] = (int)ci.size();
        if (i > 0) { ci.push_back(i - 1); va.push_back(-1.0); }
        ci.push_back(i); va.push_back(4.0);
        if (i < n - 1) { ci.push_back(i + 1); va.push_back(-1.0); }
    }
    rp[n] = (int)ci.size();
    const int nnz = (int)ci.size();
    // LU of the tridiagonal (no pivoting): L unit lower bidiagonal, U upper bidiagonal
    std::vector<double> d(n), l(n);
    d[0] = 4.0;
    for (int i = 1; i < n; ++i) { l[i] = -1.0 / d[i - 1]; d[i] = 4.0 - l[i] * -1.0; }
    std::vector<int> Lp(n + 1), Li, Up(n + 1), Ui, P(n), Q(n);
    std::vector<double> Lx, Ux;
    for (int i = 0; i < n; ++i) {
        Lp[i] = (int)Li.size();
        if (i > 0) { Li.push_back(i - 1); Lx.push_back(l[i]); }
        Li.push_back(i); Lx.push_back(1.0);
        Up[i] = (int)Ui.size();
        Ui.push_back(i); Ux.push_back(d[i]);
        if (i < n - 1) { Ui.push_back(i + 1); Ux.push_back(-1.0); }
        P[i] = i; Q[i] = i;
    }
    Lp[n] = (int)Li.size(); Up[n] = (int)Ui.size();
    cudaFree(0);
    cusolverRfHandle_t h;
    CK(cusolverRfCreate(&h));
    CK(cusolverRfSetMatrixFormat(h, CUSOLVERRF_MATRIX_FORMAT_CSR, CUSOLVERRF_UNIT_DIAGONAL_STORED_L));
    double* hv[K] = {va.data(), va.data()};
    CK(cusolverRfBatchSetupHost(K, n, nnz, rp.data(), ci.data(), hv, (int)Li.size(), Lp.data(), Li.data(), Lx.data(),
                                (int)Ui.size(), Up.data(), Ui.data(), Ux.data(), P.data(), Q.data(), h));
    CK(cusolverRfBatchAnalyze(h));
    int *drp, *dci, *dP, *dQ;
    double *dv, *dx, *dt;
    cudaMalloc(&drp, sizeof(int) * (n + 1)); cudaMalloc(&dci, sizeof(int) * nnz);
    cudaMalloc(&dP, sizeof(int) * n); cudaMalloc(&dQ, sizeof(int) * n);
    cudaMalloc(&dv, sizeof(double) * nnz * K); cudaMalloc(&dx, sizeof(double) * n * K);
    cudaMalloc(&dt, sizeof(double) * n * K * 2);
    cudaMemcpy(drp, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(dci, ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(dP, P.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dQ, Q.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
    std::vector<double> v2(va);
    for (auto& x : v2) x *= 2.0;   // scenario 1: 2A
    cudaMemcpy(dv, va.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice);
    cudaMemcpy(dv + nnz, v2.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice);
    std::vector<double> b(n * K, 1.0);
    cudaMemcpy(dx, b.data(), sizeof(double) * n * K, cudaMemcpyHostToDevice);
    double* hvd[K] = {dv, dv + nnz};
    double* hxd[K] = {dx, dx + n};
    double** dvp; double** dxp;
    cudaMalloc(&dvp, sizeof(double*) * K); cudaMalloc(&dxp, sizeof(double*) * K);
    cudaMemcpy(dvp, hvd, sizeof(hvd), cudaMemcpyHostToDevice);
    cudaMemcpy(dxp, hxd, sizeof(hxd), cudaMemcpyHostToDevice);
    const bool host_ptrs = MODE_HOST;
    CK(cusolverRfBatchResetValues(K, n, nnz, drp, dci, host_ptrs ? hvd : dvp, dP, dQ, h));
    CK(cusolverRfBatchRefactor(h));
    CK(cusolverRfBatchSolve(h, dP, dQ, 1, dt, n, host_ptrs ? hxd : dxp, n));
    CK(cudaDeviceSynchronize());
    cudaMemcpy(b.data(), dx, sizeof(double) * n * K, cudaMemcpyDeviceToHost);
    for (int k = 0; k < K; ++k) {
        // residual check: A_k x = 1
        double worst = 0;
        for (int i = 0; i < n; ++i) {
            double s = 0;
            for (int p = rp[i]; p < rp[i + 1]; ++p) s += va[p] * (k + 1) * b[k * n + ci[p]];
            worst = fmax(worst, fabs(s - 1.0));
        }
        printf("scenario %d: x0 %.6f residual %.3e\n", k, b[k * n], worst);
    }
    return 0;
}
