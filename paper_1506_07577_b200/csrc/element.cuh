// element.cuh -- per-tet element physics shared by the tet-map kernels.
//
// Displacement form: H = Du Dm^-1, F = I + H.
//   StVK: E = 1/2 (H + H^T + H^T H), S = 2 mu E + lam tr(E) I, P = F S,
//                 Psi = mu E:E + 1/2 lam tr(E)^2.
//   NH (compressible Bonet-Wood), cancellation-free invariants:
//                 delta = tr H + sigma2(H) + det H = J - 1, ln J = log1p(delta),
//                 cof F = ((1+t+sigma2) I - (1+t) H + H^2)^T,
//                 P = [mu (det H I + J H + (1+t) H^T - (H^T)^2) + lam ln J cof F] / J,
//                 Psi = 1/2 mu (2 tr H + |H|^2) - mu ln J + 1/2 lam (ln J)^2.
// Forces f_i = -W P g_i (g_i = row i-1 of Dm^-1, g_0 = -sum g_i).
// Stiffness blocks K_ij = d^2(W Psi)/dx_i dx_j, closed rank-1 forms:
//   NH   K_ij = W [mu m_ij I + c1 k_j k_i^T + lam k_i k_j^T],  k_i = F^-T g_i, c1 = mu - lam ln J
//   StVK K_ij = W [s_ij I + mu m_ij F F^T + mu h_j h_i^T + lam h_i h_j^T], h_i = F g_i, s_ij = g_i^T S g_j
#pragma once
#include <cstdint>

namespace ebb {

template <typename R>
struct TetState {
    R g[4][3];    // shape gradients g_0..g_3
    R kv[4][3];   // NH: F^-T g_i ; StVK: F g_i
    R S[3][3];    // StVK: second Piola stress
    R B[3][3];    // StVK: F F^T
    R P[3][3];    // first Piola stress
    R W, mu, lam, c1, psi, J;
};

template <typename R, int MODEL, bool WANT_K>
__device__ __forceinline__ void tet_physics(const R uu[4][3], TetState<R>& st) {
    R H[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            R s = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) s += (uu[k + 1][a] - uu[0][a]) * st.g[k + 1][b];
            H[a][b] = s;
        }
    const R mu = st.mu, lam = st.lam;
    if (MODEL == 0) {  // StVK
        R E[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                R hh = H[0][a] * H[0][b] + H[1][a] * H[1][b] + H[2][a] * H[2][b];
                E[a][b] = R(0.5) * (H[a][b] + H[b][a] + hh);
            }
        R trE = E[0][0] + E[1][1] + E[2][2];
        R EE = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                st.S[a][b] = R(2) * mu * E[a][b] + (a == b ? lam * trE : R(0));
                EE += E[a][b] * E[a][b];
            }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                st.P[a][b] = st.S[a][b] + H[a][0] * st.S[0][b] + H[a][1] * st.S[1][b] + H[a][2] * st.S[2][b];
        st.psi = mu * EE + R(0.5) * lam * trE * trE;
        st.J = R(1);
        if (WANT_K) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    st.kv[i][a] = st.g[i][a] + H[a][0] * st.g[i][0] + H[a][1] * st.g[i][1] + H[a][2] * st.g[i][2];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    R s = 0;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        s += ((a == c ? R(1) : R(0)) + H[a][c]) * ((b == c ? R(1) : R(0)) + H[b][c]);
                    st.B[a][b] = s;
                }
        }
    } else {  // NH
        R t1 = H[0][0] + H[1][1] + H[2][2];
        R H2[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) H2[a][b] = H[a][0] * H[0][b] + H[a][1] * H[1][b] + H[a][2] * H[2][b];
        R trH2 = H2[0][0] + H2[1][1] + H2[2][2];
        R s2 = R(0.5) * (t1 * t1 - trH2);
        R dH = H[0][0] * (H[1][1] * H[2][2] - H[1][2] * H[2][1]) - H[0][1] * (H[1][0] * H[2][2] - H[1][2] * H[2][0]) +
               H[0][2] * (H[1][0] * H[2][1] - H[1][1] * H[2][0]);
        R delta = t1 + s2 + dH;
        R J = R(1) + delta;
        st.J = J;
        R lnJ = log1p(delta);
        R invJ = R(1) / J;
        R ca = R(1) + t1 + s2, cb = R(1) + t1;
        R FiT[3][3];
        R HF2 = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                R cof = (a == b ? ca : R(0)) - cb * H[b][a] + H2[b][a];
                R jf = (a == b ? dH : R(0)) + J * H[a][b] + cb * H[b][a] - H2[b][a];
                st.P[a][b] = (mu * jf + lam * lnJ * cof) * invJ;
                FiT[a][b] = cof * invJ;
                HF2 += H[a][b] * H[a][b];
            }
        st.c1 = mu - lam * lnJ;
        st.psi = R(0.5) * mu * (R(2) * t1 + HF2) - mu * lnJ + R(0.5) * lam * lnJ * lnJ;
        if (WANT_K) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    st.kv[i][a] = FiT[a][0] * st.g[i][0] + FiT[a][1] * st.g[i][1] + FiT[a][2] * st.g[i][2];
        }
    }
}

// f_i = -W P g_i (i = 1..3), f_0 = -(f_1 + f_2 + f_3)
template <typename R>
__device__ __forceinline__ void tet_forces(const TetState<R>& st, R fi[4][3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) fi[0][a] = 0;
#pragma unroll
    for (int i = 1; i < 4; ++i)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            fi[i][a] = -st.W * (st.P[a][0] * st.g[i][0] + st.P[a][1] * st.g[i][1] + st.P[a][2] * st.g[i][2]);
            fi[0][a] -= fi[i][a];
        }
}

// K_ij[a][b] (closed forms above); i, j are compile-time after unrolling
template <typename R, int MODEL>
__device__ __forceinline__ void tet_block(const TetState<R>& st, int i, int j, R Kb[3][3]) {
    const R mij = st.g[i][0] * st.g[j][0] + st.g[i][1] * st.g[j][1] + st.g[i][2] * st.g[j][2];
    if (MODEL == 1) {
        const R d = st.W * st.mu * mij, cc = st.W * st.c1, cl = st.W * st.lam;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                Kb[a][b] = cc * st.kv[j][a] * st.kv[i][b] + cl * st.kv[i][a] * st.kv[j][b] + (a == b ? d : R(0));
    } else {
        R Sg[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) Sg[a] = st.S[a][0] * st.g[i][0] + st.S[a][1] * st.g[i][1] + st.S[a][2] * st.g[i][2];
        const R sij = Sg[0] * st.g[j][0] + Sg[1] * st.g[j][1] + Sg[2] * st.g[j][2];
        const R d = st.W * sij, cm = st.W * st.mu * mij, ch = st.W * st.mu, cl = st.W * st.lam;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                Kb[a][b] = cm * st.B[a][b] + ch * st.kv[j][a] * st.kv[i][b] + cl * st.kv[i][a] * st.kv[j][b] +
                           (a == b ? d : R(0));
    }
}

}  // namespace ebb
