// dist.cuh -- multi-GPU support: the 1D column-block-cyclic
// layout (block = b) and the kernels that move data between that layout and
// the replicated, globally ordered sample; NCCL is loaded at run time.
//
// Global column j lives on rank (j / b) mod P at local index
// (j / (b P)) b + j mod b; local storage keeps global order.  Panel t
// (global columns t b .. t b + bb - 1) is owned by rank t mod P.
#pragma once
#include <dlfcn.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace rq {

// ---------------------------------------------------------------------------
// layout (host + device)
// ---------------------------------------------------------------------------
__host__ __device__ inline int dist_owner(int64_t j, int b, int P) { return (int)((j / b) % P); }
__host__ __device__ inline int64_t dist_local(int64_t j, int b, int P) { return (j / ((int64_t)b * P)) * b + j % b; }
__host__ __device__ inline int64_t dist_global(int64_t lj, int b, int P, int r) {
    return ((lj / b) * P + r) * b + lj % b;
}
// number of global columns j < n owned by rank r (= first local index of r with global >= n)
__host__ __device__ inline int64_t dist_count(int64_t n, int b, int P, int r) {
    const int64_t full = n / b, rem = n % b;
    int64_t cnt = (full / P) * b;
    const int64_t extra = full % P;
    if (r < extra) cnt += b;
    if (r == extra) cnt += rem;
    return cnt;
}

// ---------------------------------------------------------------------------
// gathered (rank-major, each rank's chunk padded to cmax columns) -> global order.
// Global trailing position p (0 <= p < ncols) is global column j = j0 + p.
// ---------------------------------------------------------------------------
__global__ void dist_reorder_kernel(const double *gath, int64_t cmax, int rows, int ld, int64_t j0, int64_t ncols, int b,
                                    int P, double *out, int64_t ldo) {
    const int64_t total = ncols * rows;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e % rows, p = e / rows;
        const int64_t j = j0 + p;
        const int r = dist_owner(j, b, P);
        const int64_t c = dist_local(j, b, P) - dist_count(j0, b, P, r);
        out[row + p * ldo] = gath[row + (r * cmax + c) * ld];
    }
}

// panel broadcast pack = [tau (bbpad) | Y = strict_upper(V^T V) (bbpad^2) |
//   R11 (bbpad^2) | -T (bbpad^2, valid when the CholeskyQR2 path ran) |
//   cqr status | bb_eff | done | rank]  -- the last three are the panel
//   state after the owner's R11-diagonal stop check (iscal[1..3])
__global__ void dist_pack_kernel(const double *tau, const double *ybuf, const double *A /* R11 */, int64_t lda, int bb,
                                 int bbpad, const double *tneg, const int *status, const int *state, double *pk) {
    const int n2 = bbpad * bbpad;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bbpad + 3 * n2 + 4; e += gridDim.x * blockDim.x) {
        if (e < bbpad) pk[e] = (e < bb) ? tau[e] : 0.0;
        else if (e < bbpad + n2) pk[e] = ybuf[e - bbpad];
        else if (e < bbpad + 2 * n2) {
            const int q = e - bbpad - n2, r = q % bbpad, c = q / bbpad;
            pk[e] = (r < bb && c < bb) ? A[r + (int64_t)c * lda] : 0.0;
        } else if (e < bbpad + 3 * n2) {
            pk[e] = tneg[e - bbpad - 2 * n2];
        } else if (e == bbpad + 3 * n2) {
            pk[e] = (double)*status;
        } else {
            pk[e] = (double)state[e - (bbpad + 3 * n2 + 1)];
        }
    }
}
__global__ void dist_unpack_kernel(const double *pk, int bb, int bbpad, double *tau, double *ybuf, double *tneg,
                                   int *status, int *state) {
    const int n2 = bbpad * bbpad;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < bbpad + 3 * n2 + 4; e += gridDim.x * blockDim.x) {
        if (e < bbpad) { if (e < bb) tau[e] = pk[e]; }
        else if (e < bbpad + n2) ybuf[e - bbpad] = pk[e];
        else if (e < bbpad + 2 * n2) continue;
        else if (e < bbpad + 3 * n2) tneg[e - bbpad - 2 * n2] = pk[e];
        else if (e == bbpad + 3 * n2) *status = (int)pk[e];
        else state[e - (bbpad + 3 * n2 + 1)] = (int)pk[e];
    }
}
// Vt (bbpad x mp) from Vfull (mp x bbpad, ld ldv)
__global__ void dist_transpose_kernel(const double *vfull, int64_t ldv, int64_t mp, int bbpad, double *vt) {
    const int64_t total = mp * bbpad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e % bbpad, r = e / bbpad;
        vt[c + r * bbpad] = vfull[r + c * ldv];
    }
}
// column moves through a staging buffer: stage[:, slot[q]] = A[:, col[q]] (dir 0) or back (dir 1)
__global__ void dist_columns_kernel(double *A, int64_t lda, int64_t m, const int64_t *cols, const int *slots, int n,
                                    double *stage, int64_t lds, int dir) {
    const int64_t total = (int64_t)n * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % m, q = e / m;
        double *a = A + r + cols[q] * lda;
        double *s = stage + r + (int64_t)slots[q] * lds;
        if (dir == 0) *s = *a;
        else *a = *s;
    }
}
// replicated jpvt: jpvt[i + dst] = old jpvt[i + src] for every pair (one CTA)
__global__ void dist_jpvt_kernel(int64_t *jpvt, const int64_t *dst, const int64_t *src, const int *npairs) {
    __shared__ int64_t v[2 * 128 + 2];
    const int np = *npairs;
    for (int q = threadIdx.x; q < np; q += blockDim.x) v[q] = jpvt[src[q]];
    __syncthreads();
    for (int q = threadIdx.x; q < np; q += blockDim.x) jpvt[dst[q]] = v[q];
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the library loads without it; single-GPU use
// never touches it).  Types mirror nccl.h (NCCL 2.x ABI).
// ---------------------------------------------------------------------------
typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4, ncclUint64 = 5, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;  // optional
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                          // optional
    ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    // RQRCP_NCCL_LIB (the Python binding points it at the nvidia-nccl wheel
    // torch uses), else the soname (already mapped when torch is imported)
    const char *cands[] = {getenv("RQRCP_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *c : cands)
        if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
        api.err = "libnccl.so.2 not found (set RQRCP_NCCL_LIB)";
        return api;
    }
    auto sym = [&](const char *n) { return dlsym(h, n); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.Reduce = (decltype(api.Reduce))sym("ncclReduce");
    api.CommGetAsyncError = (decltype(api.CommGetAsyncError))sym("ncclCommGetAsyncError");
    api.CommAbort = (decltype(api.CommAbort))sym("ncclCommAbort");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.Broadcast &&
             api.AllReduce && api.Reduce && api.Send && api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
    return api;
}

}  // namespace rq
