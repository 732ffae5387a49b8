// philox.cuh -- S0 (kernel K1): the Gaussian sketch Omega ("Generate
// i.i.d Gaussian matrix Omega in N(0,1)^{(b+p) x m}").
//
// Generator (reading R-G8): element (r, c) of
// the N(0,1) matrix (seed, stream) comes from one Philox4x32-10 call (Salmon
// et al., SC'11) with key (seed lo, seed hi) and counter
// (c mod 2^32, floor(r/2), stream, c >> 32); words (w0,w1) -> u1, (w2,w3) -> u2
// as 53-bit uniforms in (0,1); Box-Muller: rows 2q / 2q+1 get
// rho cos(2 pi u2) / rho sin(2 pi u2), rho = sqrt(-2 ln u1).
// A pure function of (seed, stream, r, c): any tiling, any GPU count gives the
// same bits, so Omega is replicated across ranks with no communication.
#pragma once
#include "common.cuh"

namespace rq {

RQ_DEV uint4 philox4x32_10(uint4 x, uint2 k) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, x.x), lo0 = 0xD2511F53u * x.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, x.z), lo1 = 0xCD9E8D57u * x.z;
        x = make_uint4(hi1 ^ x.y ^ k.x, lo1, hi0 ^ x.w ^ k.y, lo0);
    }
    return x;
}

RQ_DEV double u53(uint32_t hi, uint32_t lo) {
    const uint64_t a = ((((uint64_t)hi) << 32) | lo) >> 11;
    return ((double)a + 0.5) * 0x1p-53;
}

// The normal pair (rows 2q, 2q+1) of column c.
RQ_DEV double2 normal_pair(uint64_t seed, uint32_t stream, int64_t q, int64_t c) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)((uint64_t)c & 0xFFFFFFFFu), (uint32_t)q, stream,
                                             (uint32_t)((uint64_t)c >> 32)),
                                  make_uint2((uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)));
    const double u1 = u53(w.x, w.y), u2 = u53(w.z, w.w);
    const double rho = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.141592653589793238462643383279502884 * u2;
    double s, co;
    sincos(ang, &s, &co);
    return make_double2(rho * co, rho * s);
}

// out(r, c) for r in [0,rows), c in [0,cols): element (row0+r, col0+c), column-major ld.
// One thread per (row pair, column).
__global__ void gaussian_fill_kernel(uint64_t seed, uint32_t stream, int64_t rows, int64_t cols, int64_t row0,
                                     int64_t col0, double *out, int64_t ld) {
    const int64_t first_pair = row0 >> 1;
    const int64_t last_pair = (row0 + rows - 1) >> 1;
    const int64_t npairs = last_pair - first_pair + 1;
    const int64_t total = npairs * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t qi = e % npairs, c = e / npairs;
        const int64_t q = first_pair + qi;
        const double2 z = normal_pair(seed, stream, q, col0 + c);
        const int64_t r0 = 2 * q - row0;
        if (r0 >= 0 && r0 < rows) out[r0 + c * ld] = z.x;
        if (r0 + 1 >= 0 && r0 + 1 < rows) out[r0 + 1 + c * ld] = z.y;
    }
}

// Omega^T (m x lpad, column-major ld = ldo): column r of Omega^T = row r of
// Omega, so that the sketch B = Omega A is a K-contiguous "X^T Y" product.
// Rows l..lpad-1 of Omega are zero (padding to the DMMA tile of 8).
__global__ void omega_t_kernel(uint64_t seed, int64_t l, int64_t lpad, int64_t m, double *omt, int64_t ldo) {
    const int64_t npairs = lpad / 2;
    const int64_t total = npairs * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e % m, q = e / m;  // consecutive threads: consecutive c (coalesced stores)
        double2 z = make_double2(0.0, 0.0);
        if (2 * q < l) z = normal_pair(seed, 0u, q, c);
        omt[c + (2 * q) * ldo] = z.x;
        omt[c + (2 * q + 1) * ldo] = (2 * q + 1 < l) ? z.y : 0.0;
    }
}

// Omega^T from a caller-provided Omega (l x m, ld l): transpose + zero pad.
__global__ void omega_t_from_kernel(const double *om, int64_t l, int64_t lpad, int64_t m, double *omt, int64_t ldo) {
    const int64_t total = lpad * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e % m, r = e / m;
        omt[c + r * ldo] = (r < l) ? om[r + c * l] : 0.0;
    }
}

// Omega (l x m, ld l) from Omega^T (testing hook omega_out).
__global__ void omega_from_t_kernel(const double *omt, int64_t ldo, int64_t l, int64_t m, double *om) {
    const int64_t total = l * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % l, c = e / l;
        om[r + c * l] = omt[c + r * ldo];
    }
}

__global__ void philox_words_kernel(const uint32_t *ctr, uint2 key, uint32_t *out, int64_t count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint4 w = philox4x32_10(make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]), key);
    out[4 * i] = w.x;
    out[4 * i + 1] = w.y;
    out[4 * i + 2] = w.z;
    out[4 * i + 3] = w.w;
}

}  // namespace rq
