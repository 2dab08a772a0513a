// Throughput harness for the Jacobi sweep loop (development aid): many CTAs
// (2 per SM), random 60x60 complex W in shared memory, a fixed number of
// round-robin sweeps with the production rotate_pair / neighbor hand-off.
// Variants: -DSB_NOSTORE (no write-back), -DSB_NOROT (dot products only).
// Measured on B200 (SM-cycles per round per bin, all pairs rotating): base
// 1607, no stores 816, dot products only 702 -- the round's shared-memory
// stores cost as much as everything else together.
#include "../../paper_2504_03373_b200/csrc/gsvd.cu"
#include <cstdio>
using namespace sslg;
#ifdef SB_QUAD
__constant__ unsigned char c_quad[21 * 16 * 4] = {0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,18,19,20,21,22,23,24,25,26,27,28,29,30,31,32,33,34,35,36,37,38,39,40,41,42,43,44,45,46,47,48,49,50,51,52,53,54,55,56,57,58,59,60,61,62,63,0,17,34,51,1,16,35,50,2,19,32,49,3,18,33,48,4,21,38,55,5,20,39,54,6,23,36,53,7,22,37,52,8,25,42,59,9,24,43,58,10,27,40,57,11,26,41,56,12,29,46,63,13,28,47,62,14,31,44,61,15,30,45,60,0,19,33,50,1,18,32,51,2,17,35,48,3,16,34,49,4,23,37,54,5,22,36,55,6,21,39,52,7,20,38,53,8,27,41,58,9,26,40,59,10,25,43,56,11,24,42,57,12,31,45,62,13,30,44,63,14,29,47,60,15,28,46,61,0,18,35,49,1,19,34,48,2,16,33,51,3,17,32,50,4,22,39,53,5,23,38,52,6,20,37,55,7,21,36,54,8,26,43,57,9,27,42,56,10,24,41,59,11,25,40,58,12,30,47,61,13,31,46,60,14,28,45,63,15,29,44,62,0,5,10,15,1,4,11,14,2,7,8,13,3,6,9,12,16,21,26,31,17,20,27,30,18,23,24,29,19,22,25,28,32,37,42,47,33,36,43,46,34,39,40,45,35,38,41,44,48,53,58,63,49,52,59,62,50,55,56,61,51,54,57,60,0,21,42,63,1,20,43,62,2,23,40,61,3,22,41,60,4,17,46,59,5,16,47,58,6,19,44,57,7,18,45,56,8,29,34,55,9,28,35,54,10,31,32,53,11,30,33,52,12,25,38,51,13,24,39,50,14,27,36,49,15,26,37,48,0,31,37,58,1,30,36,59,2,29,39,56,3,28,38,57,4,27,33,62,5,26,32,63,6,25,35,60,7,24,34,61,8,23,45,50,9,22,44,51,10,21,47,48,11,20,46,49,12,19,41,54,13,18,40,55,14,17,43,52,15,16,42,53,0,26,47,53,1,27,46,52,2,24,45,55,3,25,44,54,4,30,43,49,5,31,42,48,6,28,41,51,7,29,40,50,8,18,39,61,9,19,38,60,10,16,37,63,11,17,36,62,12,22,35,57,13,23,34,56,14,20,33,59,15,21,32,58,0,7,9,14,1,6,8,15,2,5,11,12,3,4,10,13,16,23,25,30,17,22,24,31,18,21,27,28,19,20,26,29,32,39,41,46,33,38,40,47,34,37,43,44,35,36,42,45,48,55,57,62,49,54,56,63,50,53,59,60,51,52,58,61,0,25,46,55,1,24,47,54,2,27,44,53,3,26,45,52,4,29,42,51,5,28,43,50,6,31,40,49,7,30,41,48,8,17,38,63,9,16,39,62,10,19,36,61,11,18,37,60,12,21,34,59,13,20,35,58,14,23,32,57,15,22,33,56,0,23,41,62,1,22,40,63,2,21,43,60,3,20,42,61,4,19,45,58,5,18,44,59,6,17,47,56,7,16,46,57,8,31,33,54,9,30,32,55,10,29,35,52,11,28,34,53,12,27,37,50,13,26,36,51,14,25,39,48,15,24,38,49,0,30,39,57,1,31,38,56,2,28,37,59,3,29,36,58,4,26,35,61,5,27,34,60,6,24,33,63,7,25,32,62,8,22,47,49,9,23,46,48,10,20,45,51,11,21,44,50,12,18,43,53,13,19,42,52,14,16,41,55,15,17,40,54,0,6,11,13,1,7,10,12,2,4,9,15,3,5,8,14,16,22,27,29,17,23,26,28,18,20,25,31,19,21,24,30,32,38,43,45,33,39,42,44,34,36,41,47,35,37,40,46,48,54,59,61,49,55,58,60,50,52,57,63,51,53,56,62,0,29,38,59,1,28,39,58,2,31,36,57,3,30,37,56,4,25,34,63,5,24,35,62,6,27,32,61,7,26,33,60,8,21,46,51,9,20,47,50,10,23,44,49,11,22,45,48,12,17,42,55,13,16,43,54,14,19,40,53,15,18,41,52,0,27,45,54,1,26,44,55,2,25,47,52,3,24,46,53,4,31,41,50,5,30,40,51,6,29,43,48,7,28,42,49,8,19,37,62,9,18,36,63,10,17,39,60,11,16,38,61,12,23,33,58,13,22,32,59,14,21,35,56,15,20,34,57,0,22,43,61,1,23,42,60,2,20,41,63,3,21,40,62,4,18,47,57,5,19,46,56,6,16,45,59,7,17,44,58,8,30,35,53,9,31,34,52,10,28,33,55,11,29,32,54,12,26,39,49,13,27,38,48,14,24,37,51,15,25,36,50,0,4,8,12,1,5,9,13,2,6,10,14,3,7,11,15,16,20,24,28,17,21,25,29,18,22,26,30,19,23,27,31,32,36,40,44,33,37,41,45,34,38,42,46,35,39,43,47,48,52,56,60,49,53,57,61,50,54,58,62,51,55,59,63,0,20,40,60,1,21,41,61,2,22,42,62,3,23,43,63,4,16,44,56,5,17,45,57,6,18,46,58,7,19,47,59,8,28,32,52,9,29,33,53,10,30,34,54,11,31,35,55,12,24,36,48,13,25,37,49,14,26,38,50,15,27,39,51,0,28,36,56,1,29,37,57,2,30,38,58,3,31,39,59,4,24,32,60,5,25,33,61,6,26,34,62,7,27,35,63,8,20,44,48,9,21,45,49,10,22,46,50,11,23,47,51,12,16,40,52,13,17,41,53,14,18,42,54,15,19,43,55,0,24,44,52,1,25,45,53,2,26,46,54,3,27,47,55,4,28,40,48,5,29,41,49,6,30,42,50,7,31,43,51,8,16,36,60,9,17,37,61,10,18,38,62,11,19,39,63,12,20,32,56,13,21,33,57,14,22,34,58,15,23,35,59,0,16,32,48,1,17,33,49,2,18,34,50,3,19,35,51,4,20,36,52,5,21,37,53,6,22,38,54,7,23,39,55,8,24,40,56,9,25,41,57,10,26,42,58,11,27,43,59,12,28,44,60,13,29,45,61,14,30,46,62,15,31,47,63};

// two disjoint pairs of a 16-lane group's four register columns, split
// rotation parameters (lanes 0-7 pair A, 8-15 pair B) swapped by shuffles
template <int RPL, int GL, int A0, int B0, int A1, int B1>
__device__ __forceinline__ int qrot2(double2 (&C)[4][RPL], double (&n)[4], unsigned& dirty, int js) {
    double ax = 0, ay = 0, bx = 0, by = 0;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
        const double2 p0 = C[A0][u], q0 = C[B0][u], p1 = C[A1][u], q1 = C[B1][u];
        ax = fma(p0.x, q0.x, fma(p0.y, q0.y, ax));
        ay = fma(p0.x, q0.y, fma(-p0.y, q0.x, ay));
        bx = fma(p1.x, q1.x, fma(p1.y, q1.y, bx));
        by = fma(p1.x, q1.y, fma(-p1.y, q1.x, by));
    }
    constexpr int H = GL / 2;
    const unsigned mask = group_mask<GL>();
    const bool lo = js < H;
    double mx = lo ? ax : bx, my = lo ? ay : by;
    {
        const double sx = lo ? bx : ax, sy = lo ? by : ay;
        mx += __shfl_xor_sync(mask, sx, H);
        my += __shfl_xor_sync(mask, sy, H);
    }
#pragma unroll
    for (int o = H / 2; o > 0; o >>= 1) {
        mx += __shfl_xor_sync(mask, mx, o);
        my += __shfl_xor_sync(mask, my, o);
    }
    double cp = lo ? n[A0] : n[A1], cq = lo ? n[B0] : n[B1];
    const double M = fma(mx, mx, my * my);
    const bool on = !(cp <= 0.0 || cq <= 0.0 || M <= 1e-28 * cp * cq);
    JRot r;
    r.c = 1.0;
    r.sn = r.alx = r.aly = r.bex = r.bey = 0.0;
    if (on) {
        r = jrot(mx, my, cp, cq);
        const double np = r.c * r.c * cp - r.cs2 + r.sn * r.sn * cq;
        cq = r.sn * r.sn * cp + r.cs2 + r.c * r.c * cq;
        cp = np;
    }
    JRot o;
    o.c = __shfl_xor_sync(mask, r.c, H);
    o.sn = __shfl_xor_sync(mask, r.sn, H);
    o.alx = __shfl_xor_sync(mask, r.alx, H);
    o.aly = __shfl_xor_sync(mask, r.aly, H);
    o.bex = __shfl_xor_sync(mask, r.bex, H);
    o.bey = __shfl_xor_sync(mask, r.bey, H);
    const double ocp = __shfl_xor_sync(mask, cp, H), ocq = __shfl_xor_sync(mask, cq, H);
    const bool oon = __shfl_xor_sync(mask, (int)on, H) != 0;
    const bool aon = lo ? on : oon, bon = lo ? oon : on;
    int cnt = 0;
    if (aon) {
        const double c = lo ? r.c : o.c, sn = lo ? r.sn : o.sn, alx = lo ? r.alx : o.alx, aly = lo ? r.aly : o.aly;
        const double bex = lo ? r.bex : o.bex, bey = lo ? r.bey : o.bey;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
            const double2 x = C[A0][u], y = C[B0][u];
            C[A0][u].x = fma(c, x.x, fma(-alx, y.x, aly * y.y));
            C[A0][u].y = fma(c, x.y, fma(-alx, y.y, -aly * y.x));
            C[B0][u].x = fma(sn, x.x, fma(bex, y.x, -bey * y.y));
            C[B0][u].y = fma(sn, x.y, fma(bex, y.y, bey * y.x));
        }
        n[A0] = lo ? cp : ocp;
        n[B0] = lo ? cq : ocq;
        dirty |= (1u << A0) | (1u << B0);
        ++cnt;
    }
    if (bon) {
        const double c = lo ? o.c : r.c, sn = lo ? o.sn : r.sn, alx = lo ? o.alx : r.alx, aly = lo ? o.aly : r.aly;
        const double bex = lo ? o.bex : r.bex, bey = lo ? o.bey : r.bey;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
            const double2 x = C[A1][u], y = C[B1][u];
            C[A1][u].x = fma(c, x.x, fma(-alx, y.x, aly * y.y));
            C[A1][u].y = fma(c, x.y, fma(-alx, y.y, -aly * y.x));
            C[B1][u].x = fma(sn, x.x, fma(bex, y.x, -bey * y.y));
            C[B1][u].y = fma(sn, x.y, fma(bex, y.y, bey * y.x));
        }
        n[A1] = lo ? ocp : cp;
        n[B1] = lo ? ocq : cq;
        dirty |= (1u << A1) | (1u << B1);
        ++cnt;
    }
    return cnt;
}
#endif
__global__ void __launch_bounds__(256, 2) sweep_bench(double2* out, int m, int sweeps, long long* clk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    __shared__ double cn[kMaxM];
    const int tid = threadIdx.x;
    for (int e = tid; e < m * m; e += blockDim.x) {
        unsigned h = (unsigned)(e * 2654435761u) ^ (unsigned)(blockIdx.x * 40503u);
        W[e] = make_double2((h & 0xffff) / 65536.0 - 0.5, ((h >> 16) & 0xffff) / 65536.0 - 0.5);
    }
    if (tid < m) cn[tid] = 0;
    __syncthreads();
    const int g = tid / kLPP, s = tid % kLPP;
    const int n_even = (m + 1) & ~1, npairs = n_even / 2;
    for (int j = g * 2; j < g * 2 + 2 && j < m; ++j) {
        double v = 0;
        for (int u = 0; u < kRows; ++u) { const int row = s + u * kLPP; if (row < m) v += cnorm(W[j * m + row]); }
        v = group_sum<kLPP>(v);
        if (s == 0) cn[j] = v;
    }
    __syncthreads();
    long long t0 = clock64();
    double mymax = 0;
    int rots = 0;
#ifdef SB_QUAD
    {
        constexpr int GL = 16, RPL = 4;
        const int qg = tid / GL, js = tid % GL;
        for (int sw = 0; sw < sweeps; ++sw) {
            for (int r = 0; r < 21; ++r) {
                int cols[4];
                double2 C[4][RPL];
                double n[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    cols[i] = c_quad[(r * 16 + qg) * 4 + i];
#pragma unroll
                    for (int u = 0; u < RPL; ++u) {
                        const int row = js + GL * u;
                        C[i][u] = (cols[i] < m && row < m) ? W[cols[i] * m + row] : make_double2(0, 0);
                    }
                    n[i] = cols[i] < m ? cn[cols[i]] : 0.0;
                }
                unsigned dirty = 0;
                rots += qrot2<RPL, GL, 0, 1, 2, 3>(C, n, dirty, js);
                rots += qrot2<RPL, GL, 0, 2, 1, 3>(C, n, dirty, js);
                rots += qrot2<RPL, GL, 0, 3, 1, 2>(C, n, dirty, js);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if ((dirty >> i) & 1u) {
#pragma unroll
                        for (int u = 0; u < RPL; ++u) {
                            const int row = js + GL * u;
                            if (row < m) W[cols[i] * m + row] = C[i][u];
                        }
                        if (js == 0) cn[cols[i]] = n[i];
                    }
                __syncthreads();
            }
        }
    }
#elif defined(SB_HALVE)
    int n2 = 2;
    while (n2 < m) n2 <<= 1;
    const bool gact = g < n2 / 2;
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int S = n2; S >= 2; S >>= 1) {
            const int h = S >> 1;
            const int kset = g / h, gi = g % h;
            const int ia = kset * S + gi;
            int ib = kset * S + h + gi;
            double2 Aa[kRows], Bb[kRows];
            double ca = 0.0, cb = 0.0;
            bool adirty = false;
            if (gact) {
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    Aa[u] = (row < m && ia < m) ? W[ia * m + row] : make_double2(0, 0);
                    Bb[u] = (row < m && ib < m) ? W[ib * m + row] : make_double2(0, 0);
                }
                ca = ia < m ? cn[ia] : 0.0;
                cb = ib < m ? cn[ib] : 0.0;
            }
            for (int rnd = 0; rnd < h; ++rnd) {
                if (gact && ia < m && ib < m) {
                    if (rotate_pair<kRows, kLPP>(Aa, Bb, ca, cb, 0.0, s, m, mymax)) {
                        adirty = true;
                        ++rots;
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            if (row < m) W[ib * m + row] = Bb[u];
                        }
                        if (s == 0) cn[ib] = cb;
                    }
                }
                if (rnd + 1 < h) {
                    __syncthreads();
                    ib = kset * S + h + ((gi + rnd + 1) & (h - 1));
                    if (gact) {
#pragma unroll
                        for (int u = 0; u < kRows; ++u) {
                            const int row = s + u * kLPP;
                            Bb[u] = (row < m && ib < m) ? W[ib * m + row] : make_double2(0, 0);
                        }
                        cb = ib < m ? cn[ib] : 0.0;
                    }
                }
            }
            if (gact && adirty) {
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    if (row < m) W[ia * m + row] = Aa[u];
                }
                if (s == 0) cn[ia] = ca;
            }
            __syncthreads();
        }
    }
#else
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int r = 0; r < n_even - 1; ++r) {
            if (g < npairs) {
                int p, q;
                rr_pair(r, g, n_even, p, q);
                double2 P[kRows], Q[kRows];
#pragma unroll
                for (int u = 0; u < kRows; ++u) {
                    const int row = s + u * kLPP;
                    P[u] = row < m ? W[p * m + row] : make_double2(0, 0);
                    Q[u] = row < m ? W[q * m + row] : make_double2(0, 0);
                }
                double cp = cn[p], cq = cn[q];
#ifdef SB_NOROT
                double d0 = 0;
                for (int u = 0; u < kRows; ++u) d0 = fma(P[u].x, Q[u].x, fma(P[u].y, Q[u].y, d0));
                d0 = group_sum<kLPP>(d0);
                rots += d0 > 1e300;
#else
                if (rotate_pair<kRows, kLPP>(P, Q, cp, cq, 0.0, s, m, mymax)) {
                    ++rots;
#ifndef SB_NOSTORE
#pragma unroll
                    for (int u = 0; u < kRows; ++u) {
                        const int row = s + u * kLPP;
                        if (row < m) {
                            W[p * m + row] = P[u];
                            W[q * m + row] = Q[u];
                        }
                    }
                    if (s == 0) { cn[p] = cp; cn[q] = cq; }
#endif
                }
#endif
            }
            __syncthreads();
        }
    }
#endif
    long long t1 = clock64();
    if (tid == 0) atomicAdd((unsigned long long*)clk, (unsigned long long)(t1 - t0));
    if (tid == 0) out[blockIdx.x] = make_double2(W[0].x + rots, mymax);
}

// 16-lane pair groups (4 rows per lane), 512 threads: the one-bin-per-SM
// layout (MINB = 1, shared memory padded so only one CTA fits) against two
// such CTAs per SM (MINB = 2, 64 registers)
template <int MINB, int L = 16, int R = 4, int NT = 512>
__global__ void __launch_bounds__(NT, MINB) sweep_bench16(double2* out, int m, int sweeps, long long* clk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* W = reinterpret_cast<double2*>(smem_raw);
    __shared__ double cn[kMaxM];
    const int tid = threadIdx.x;
    for (int e = tid; e < m * m; e += blockDim.x) {
        unsigned h = (unsigned)(e * 2654435761u) ^ (unsigned)(blockIdx.x * 40503u);
        W[e] = make_double2((h & 0xffff) / 65536.0 - 0.5, ((h >> 16) & 0xffff) / 65536.0 - 0.5);
    }
    if (tid < m) cn[tid] = 0;
    __syncthreads();
    const int g = tid / L, s = tid % L;
    const int n_even = (m + 1) & ~1, npairs = n_even / 2;
    for (int j = g * 2; j < g * 2 + 2 && j < m; ++j) {
        double v = 0;
        for (int u = 0; u < R; ++u) { const int row = s + u * L; if (row < m) v += cnorm(W[j * m + row]); }
        v = group_sum<L>(v);
        if (s == 0) cn[j] = v;
    }
    __syncthreads();
    long long t0 = clock64();
    double mymax = 0;
    int rots = 0;
    for (int sw = 0; sw < sweeps; ++sw) {
        for (int r = 0; r < n_even - 1; ++r) {
            if (g < npairs) {
                int p, q;
                rr_pair(r, g, n_even, p, q);
                double2 P[R], Q[R];
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    const int row = s + u * L;
                    P[u] = row < m ? W[p * m + row] : make_double2(0, 0);
                    Q[u] = row < m ? W[q * m + row] : make_double2(0, 0);
                }
                double cp = cn[p], cq = cn[q];
                if (rotate_pair<R, L>(P, Q, cp, cq, 0.0, s, m, mymax)) {
                    ++rots;
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int row = s + u * L;
                        if (row < m) {
                            W[p * m + row] = P[u];
                            W[q * m + row] = Q[u];
                        }
                    }
                    if (s == 0) { cn[p] = cp; cn[q] = cq; }
                }
            }
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (tid == 0) atomicAdd((unsigned long long*)clk, (unsigned long long)(t1 - t0));
    if (tid == 0) out[blockIdx.x] = make_double2(W[0].x + rots, mymax);
}
template <int MINB, int L = 16, int R = 4, int NT = 512>
void run16(int m, int sweeps, const char* name, int smem_force = 0) {
    const int ctas = 148 * 2 * 4;
    double2* out; long long* clk;
    cudaMalloc(&out, ctas * sizeof(double2)); cudaMalloc(&clk, 8);
    const int smem = smem_force ? smem_force : (MINB == 1 ? 150 * 1024 : m * m * 16);
    cudaFuncSetAttribute(sweep_bench16<MINB, L, R, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(clk, 0, 8);
        cudaEventRecord(a);
        sweep_bench16<MINB, L, R, NT><<<ctas, NT, smem>>>(out, m, sweeps, clk);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double rounds = (double)sweeps * (m - 1);
        printf("%-12s %.3f ms  SM-cycles/round-of-one-bin %.0f (%s)\n", name, ms,
               ms * 1e-3 * 1.965e9 * 148 / (ctas * rounds), cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
#ifdef SB_L16
    run16<1>(60, 4, "L16x1");
    run16<2>(60, 4, "L16x2");
    return 0;
#endif
#ifdef SB_L4
    // 4-lane groups, 16 rows per lane, 128 threads: 2 CTAs per SM (the
    // production scratch would allow no more) and 3
    run16<2, 4, 16, 128>(60, 4, "L4x2", 100 * 1024);
    run16<3, 4, 16, 128>(60, 4, "L4x3", 70 * 1024);
    run16<2, 8, 8, 256>(60, 4, "L8x2(base)", 100 * 1024);
    return 0;
#endif
    const int m = 60, sweeps = 4, ctas = 148 * 2 * 4;
    double2* out; long long* clk;
    cudaMalloc(&out, ctas * sizeof(double2)); cudaMalloc(&clk, 8);
    const int smem = m * m * 16;
    cudaFuncSetAttribute(sweep_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(clk, 0, 8);
        cudaEventRecord(a);
        sweep_bench<<<ctas, 256, smem>>>(out, m, sweeps, clk);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
#ifdef SB_QUAD
        const double rounds = (double)sweeps * 59.0 * (1770.0 / 2016.0) * 0 + sweeps * 59.0;  // per round-of-the-circle-method equivalent
#else
        const double rounds = (double)sweeps * (m - 1);
#endif
        printf("%-12s %.3f ms  per-CTA cycles/round %.0f  SM-cycles/round-of-one-bin %.0f (%s)\n", VARIANT, ms,
               (double)c / ctas / rounds, ms * 1e-3 * 1.965e9 * 148 / (ctas * rounds), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
