// seg_common.cuh -- compact per-instance element state shared by the
// segmented element maps (seg_map.cu: owner tiles; chunk_map.cu: tet chunks
// with forward messages).  Phase 1 writes one instance's state column into
// shared memory (SoA, NT columns); phase 2 rebuilds the 3x3 blocks K_ij of
// an edge row from the states of its contributing (instance, i, j).
#pragma once
#include <cstdint>

#include "../../include/ebb.h"
#include "element.cuh"

namespace ebb {

// ------------------------------------------------------------------ state
template <int MODEL>
struct SegState;
template <>
struct SegState<EBB_NH> {   // [k 12][W mu m_p 10][W c1][W lam][f 12]
    static constexpr int KV = 0, CM = 12, C1 = 22, CL = 23, F = 24, SW = 36;
};
template <>
struct SegState<EBB_STVK> { // [h 12][W s_p 10][W mu m_p 10][B 6][W mu][W lam][f 12]
    static constexpr int KV = 0, WS = 12, WM = 22, B = 32, CH = 38, CL = 39, F = 40, SW = 52;
};

// pair order: off-diagonal (0,1) (0,2) (0,3) (1,2) (1,3) (2,3), diagonal (0,0)..(3,3)
__host__ __device__ constexpr int pair_i(int p) { return p < 3 ? 0 : p < 5 ? 1 : p < 6 ? 2 : p - 6; }
__host__ __device__ constexpr int pair_j(int p) { return p < 3 ? p + 1 : p < 5 ? p - 1 : p < 6 ? 3 : p - 6; }

template <typename R>
struct SegIn {
    R uu[4][3];
    R g[3][3];
    R W, mu, lam;
};

template <typename R>
__device__ __forceinline__ void seg_load(uint32_t t, uint4 v, uint64_t nt, const R* __restrict__ u,
                                         const R* __restrict__ Dminv, const R* __restrict__ Wt,
                                         const R* __restrict__ mu_t, const R* __restrict__ lam_t, SegIn<R>& in) {
    if (t == 0xFFFFFFFFu) return;
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#ifdef SEG_NO_GATHER   // measurement-only build: no u gathers (wrong results)
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a) in.uu[k][a] = R(1e-4) * (R)((vv[k] + a) & 15);
#else
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a) in.uu[k][a] = __ldg(u + 3ull * vv[k] + a);
#endif
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) in.g[r][c] = __ldg(Dminv + (uint64_t)(3 * r + c) * nt + t);
    in.W = __ldg(Wt + t);
    in.mu = __ldg(mu_t + t);
    in.lam = __ldg(lam_t + t);
}

// Adds one stored off-diagonal block (entry = oi | oj << 13 | pair << 26 with
// oi = 3 i NT + lr, oj = 3 j NT + lr the word offsets of k_i, k_j in the state):
//   NH   K_ij = W [ mu m_ij I + c1 k_j k_i^T + lam k_i k_j^T ]
//   StVK K_ij = W [ s_ij I + mu (m_ij F F^T + h_j h_i^T) + lam h_i h_j^T ]
// as K[a][b] += (W c1 k_j)[a] k_i[b] + (W lam k_i)[a] k_j[b] (+ the I and F F^T terms).
template <typename R, int MODEL, int NT>
__device__ __forceinline__ void seg_block(const R* __restrict__ st, uint32_t ent, R acc[9]) {
    using G = SegState<MODEL>;
    // entry = word offsets of k_i[0] and k_j[0] in the state, and the pair
    const uint32_t oi = ent & 0x1FFFu, oj = (ent >> 13) & 0x1FFFu, p = ent >> 26, lr = oi % NT;
    const R* si = st + G::KV * NT + oi;
    const R* sj = st + G::KV * NT + oj;
    const R ki[3] = {si[0], si[NT], si[2 * NT]};
    const R kj[3] = {sj[0], sj[NT], sj[2 * NT]};
    R ca, cb, cc;
    if constexpr (MODEL == EBB_NH) {
        ca = st[(G::CM + p) * NT + lr];
        cb = st[G::C1 * NT + lr];
        cc = st[G::CL * NT + lr];
    } else {
        ca = st[(G::WS + p) * NT + lr];
        cb = st[G::CH * NT + lr];
        cc = st[G::CL * NT + lr];
    }
    const R uj[3] = {cb * kj[0], cb * kj[1], cb * kj[2]};
    const R wi[3] = {cc * ki[0], cc * ki[1], cc * ki[2]};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            R v = fma(uj[a], ki[b], acc[3 * a + b]);
            acc[3 * a + b] = fma(wi[a], kj[b], v);
        }
    acc[0] += ca;
    acc[4] += ca;
    acc[8] += ca;
    if constexpr (MODEL != EBB_NH) {
        const R cd = st[(G::WM + p) * NT + lr];
        constexpr int bidx[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) acc[3 * a + b] = fma(cd, st[(G::B + bidx[a][b]) * NT + lr], acc[3 * a + b]);
    }
}

// Adds one diagonal block K_ii (symmetric: 6 unique, acc = 00 01 02 11 12 22):
//   NH   K_ii = W [ mu m_ii I + (c1 + lam) k_i k_i^T ]
//   StVK K_ii = W [ s_ii I + mu m_ii F F^T + (mu + lam) h_i h_i^T ]
template <typename R, int MODEL, int NT>
__device__ __forceinline__ void seg_diag(const R* __restrict__ st, uint32_t ent, R acc[6]) {
    using G = SegState<MODEL>;
    const uint32_t oi = ent & 0x1FFFu, p = ent >> 26, lr = oi % NT;
    const R* si = st + G::KV * NT + oi;
    const R k[3] = {si[0], si[NT], si[2 * NT]};
    R ca, sc;
    if constexpr (MODEL == EBB_NH) {
        ca = st[(G::CM + p) * NT + lr];
        sc = st[G::C1 * NT + lr] + st[G::CL * NT + lr];
    } else {
        ca = st[(G::WS + p) * NT + lr];
        sc = st[G::CH * NT + lr] + st[G::CL * NT + lr];
    }
    const R v[3] = {sc * k[0], sc * k[1], sc * k[2]};
    acc[0] = fma(v[0], k[0], acc[0] + ca);
    acc[1] = fma(v[0], k[1], acc[1]);
    acc[2] = fma(v[0], k[2], acc[2]);
    acc[3] = fma(v[1], k[1], acc[3] + ca);
    acc[4] = fma(v[1], k[2], acc[4]);
    acc[5] = fma(v[2], k[2], acc[5] + ca);
    if constexpr (MODEL != EBB_NH) {
        const R cd = st[(G::WM + p) * NT + lr];
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[q] = fma(cd, st[(G::B + q) * NT + lr], acc[q]);
    }
}


// Phase 1 epilogue: one instance's compact state into its shared-memory
// column sr (sr = st + slot; word w of the state at sr[w * NT]).
template <typename R, int MODEL, int NT>
__device__ __forceinline__ void seg_put_state(const TetState<R>& ts, const R fi[4][3], R* sr) {
    using G = SegState<MODEL>;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            sr[(G::KV + 3 * i + a) * NT] = ts.kv[i][a];
            sr[(G::F + 3 * i + a) * NT] = fi[i][a];
        }
#pragma unroll
    for (int p = 0; p < 10; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const R mij = ts.g[i][0] * ts.g[j][0] + ts.g[i][1] * ts.g[j][1] + ts.g[i][2] * ts.g[j][2];
        if constexpr (MODEL == EBB_NH) {
            sr[(SegState<EBB_NH>::CM + p) * NT] = ts.W * ts.mu * mij;
        } else {
            R Sg[3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
                Sg[a] = ts.S[a][0] * ts.g[i][0] + ts.S[a][1] * ts.g[i][1] + ts.S[a][2] * ts.g[i][2];
            sr[(SegState<EBB_STVK>::WS + p) * NT] = ts.W * (Sg[0] * ts.g[j][0] + Sg[1] * ts.g[j][1] + Sg[2] * ts.g[j][2]);
            sr[(SegState<EBB_STVK>::WM + p) * NT] = ts.W * ts.mu * mij;
        }
    }
    if constexpr (MODEL == EBB_NH) {
        sr[SegState<EBB_NH>::C1 * NT] = ts.W * ts.c1;
        sr[SegState<EBB_NH>::CL * NT] = ts.W * ts.lam;
    } else {
        constexpr int B = SegState<EBB_STVK>::B;
        sr[(B + 0) * NT] = ts.B[0][0];
        sr[(B + 1) * NT] = ts.B[0][1];
        sr[(B + 2) * NT] = ts.B[0][2];
        sr[(B + 3) * NT] = ts.B[1][1];
        sr[(B + 4) * NT] = ts.B[1][2];
        sr[(B + 5) * NT] = ts.B[2][2];
        sr[SegState<EBB_STVK>::CH * NT] = ts.W * ts.mu;
        sr[SegState<EBB_STVK>::CL * NT] = ts.W * ts.lam;
    }
}

}  // namespace ebb
