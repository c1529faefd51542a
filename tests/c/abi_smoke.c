/* C-only use of the boundary (include/hmmscan.h, libhmmscan.so): no Python, no torch.  A 4-state
 * sticky HMM with deterministic pseudo-observations, T = 100003 steps; checks the paper's invariants
 * on the results (every smoothed / filtered row a distribution, smoothed_{T-1} = filtered_{T-1}
 * (Eq. 14 at t = T-1), log p(x*, y) <= log Z, the path inside [0, D)).  Parity with the fp64 oracle
 * is the Python suite's job; this program shows the library is callable from C as declared.
 * Exit code 0 = pass. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include "hmmscan.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("cuda: %s\n", cudaGetErrorString(e_)); return 2; } } while (0)

int main(void) {
    const int D = 4;
    const int64_t T = 100003;
    float lp[4], la[16];
    for (int i = 0; i < D; i++) {
        lp[i] = logf(0.25f);
        for (int j = 0; j < D; j++) la[i * D + j] = logf(i == j ? 0.91f : 0.03f);
    }
    float* ll = (float*)malloc(sizeof(float) * T * D);
    unsigned s = 12345u;
    for (int64_t t = 0; t < T; t++) {
        s = s * 1664525u + 1013904223u;
        const int obs = (int)((s >> 16) % D);
        for (int d = 0; d < D; d++) ll[t * D + d] = logf(d == obs ? 0.7f : 0.1f);
    }
    float *dlp, *dla, *dll, *dfilt, *dsm;
    double *dlz, *dlpr;
    int32_t *dinfo, *dvinfo, *dpath;
    CK(cudaMalloc((void**)&dlp, sizeof lp));
    CK(cudaMalloc((void**)&dla, sizeof la));
    CK(cudaMalloc((void**)&dll, sizeof(float) * T * D));
    CK(cudaMalloc((void**)&dfilt, sizeof(float) * T * D));
    CK(cudaMalloc((void**)&dsm, sizeof(float) * T * D));
    CK(cudaMalloc((void**)&dpath, sizeof(int32_t) * T));
    CK(cudaMalloc((void**)&dlz, sizeof(double)));
    CK(cudaMalloc((void**)&dlpr, sizeof(double)));
    CK(cudaMalloc((void**)&dinfo, sizeof(int32_t)));
    CK(cudaMalloc((void**)&dvinfo, sizeof(int32_t)));
    CK(cudaMemcpy(dlp, lp, sizeof lp, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dla, la, sizeof la, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dll, ll, sizeof(float) * T * D, cudaMemcpyHostToDevice));
    size_t ws0 = hmm_workspace_size(HMM_OP_SMOOTH, D, T, 1), ws1 = hmm_workspace_size(HMM_OP_VITERBI, D, T, 1);
    size_t wsb = ws0 > ws1 ? ws0 : ws1;
    if (wsb == 0) { printf("workspace size 0\n"); return 1; }
    void* ws;
    CK(cudaMalloc(&ws, wsb));
    CK(cudaMemset(ws, 0, wsb));  /* zero-filled once; the library leaves it zeroed */
    hmm_status_t st = hmm_smooth(D, T, dlp, dla, dll, dfilt, dsm, dlz, dinfo, ws, wsb, NULL);
    if (st != HMM_SUCCESS) { printf("hmm_smooth: %s\n", hmm_status_string(st)); return 1; }
    st = hmm_viterbi(D, T, dlp, dla, dll, dpath, dlpr, dvinfo, ws, wsb, NULL);
    if (st != HMM_SUCCESS) { printf("hmm_viterbi: %s\n", hmm_status_string(st)); return 1; }
    CK(cudaDeviceSynchronize());
    float* filt = (float*)malloc(sizeof(float) * T * D);
    float* sm = (float*)malloc(sizeof(float) * T * D);
    int32_t* path = (int32_t*)malloc(sizeof(int32_t) * T);
    double lz, lpr;
    int32_t info, vinfo;
    CK(cudaMemcpy(filt, dfilt, sizeof(float) * T * D, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sm, dsm, sizeof(float) * T * D, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(path, dpath, sizeof(int32_t) * T, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&lz, dlz, sizeof lz, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&lpr, dlpr, sizeof lpr, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&info, dinfo, sizeof info, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&vinfo, dvinfo, sizeof vinfo, cudaMemcpyDeviceToHost));
    double worst = 0.0;
    for (int64_t t = 0; t < T; t++) {
        double a = 0.0, b = 0.0;
        for (int d = 0; d < D; d++) { a += filt[t * D + d]; b += sm[t * D + d]; }
        if (fabs(a - 1.0) > worst) worst = fabs(a - 1.0);
        if (fabs(b - 1.0) > worst) worst = fabs(b - 1.0);
    }
    double last = 0.0;
    for (int d = 0; d < D; d++) last = fmax(last, fabs((double)filt[(T - 1) * D + d] - sm[(T - 1) * D + d]));
    int bad_path = 0;
    for (int64_t t = 0; t < T; t++) bad_path += (path[t] < 0 || path[t] >= D);
    printf("%s | info %d/%d  log Z %.6f  log p(x*,y) %.6f  max |row sum - 1| %.2e  |sm_T-1 - filt_T-1| %.2e\n",
           hmm_version(), info, vinfo, lz, lpr, worst, last);
    const int ok = info == 0 && vinfo == 0 && worst < 1e-5 && last < 1e-5 && bad_path == 0 && lpr <= lz &&
                   isfinite(lz) && isfinite(lpr);
    return ok ? 0 : 1;
}
