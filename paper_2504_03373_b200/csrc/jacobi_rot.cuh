// The Jacobi rotation of one column pair (reference gsvd.cpp:642-672),
// shared by the CTA solver (gsvd.cu) and the warp solver of small arrays
// (small.cu).
#pragma once
#include "common.cuh"

namespace sslg {

// Rotation of one pair (gsvd.cpp:642-672) in closed form.  With D = cq - cp,
// M = |a_pq|^2 and q = sqrt(4M + D^2), the reference's
//   tau = D / (2|a_pq|), t = sgn(tau) / (|tau| + sqrt(1 + tau^2)),
//   c = 1 / sqrt(1 + t^2), s = t c
// are c = sqrt((q + |D|) / (2q)) and s = sgn(D) sqrt(2M / (q (q + |D|))):
// two dependent rsqrt instead of four.
struct JRot {
    double c, sn, alx, aly, bex, bey, cs2;
    bool on;
};

__device__ __forceinline__ JRot jrot(double dx, double dy, double cp, double cq) {
    JRot r;
    r.on = true;
    const double M = fma(dx, dx, dy * dy);
    const double D = cq - cp;
    const double aD = fabs(D);
    const double iM = fast_rsqrt(M);  // 1 / |a_pq|
    const double phx = dx * iM, phy = dy * iM;
    double c, sn;
    if (__builtin_expect(aD < 1e150 && M < 1e300, 1)) {
        const double q2 = fma(D, D, 4.0 * M);
        const double q = q2 * fast_rsqrt(q2);
        const double iv = fast_rsqrt(q * (q + aD));
        c = (q + aD) * iv * 0.70710678118654752440;
        sn = copysign(1.41421356237309504880 * (M * iM) * iv, D);
    } else {  // tau^2 would overflow: the reference's formula, t ~ 1 / (2|tau|)
        const double tau = D * (0.5 * iM);
        const double t = copysign(0.5 / fabs(tau), tau);
        c = fast_rsqrt(fma(t, t, 1.0));
        sn = t * c;
    }
    r.c = c;
    r.sn = sn;
    r.alx = sn * phx;
    r.aly = -sn * phy;
    r.bex = c * phx;
    r.bey = -c * phy;
    r.cs2 = 2.0 * c * sn * (M * iM);
    return r;
}
template <int RPL>
__device__ __forceinline__ void japply(double2 (&P)[RPL], double2 (&Q)[RPL], const JRot& r, double& cp, double& cq) {
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
        const double2 x = P[u], y = Q[u];
        P[u].x = fma(r.c, x.x, fma(-r.alx, y.x, r.aly * y.y));
        P[u].y = fma(r.c, x.y, fma(-r.alx, y.y, -r.aly * y.x));
        Q[u].x = fma(r.sn, x.x, fma(r.bex, y.x, -r.bey * y.y));
        Q[u].y = fma(r.sn, x.y, fma(r.bex, y.y, r.bey * y.x));
    }
    const double np = r.c * r.c * cp - r.cs2 + r.sn * r.sn * cq;
    cq = r.sn * r.sn * cp + r.cs2 + r.c * r.c * cq;
    cp = np;
}

// One Jacobi pair in registers (gsvd.cpp:642-672): P is the lower-index
// column.  Returns whether a rotation was applied.
template <int R, int L>
__device__ __forceinline__ bool rotate_pair(double2 (&P)[R], double2 (&Q)[R], double& cp, double& cq, double drop,
                                            int s, int m, double& maxrel, double tol2) {
    double d0x = 0, d0y = 0, d1x = 0, d1y = 0;
#pragma unroll
    for (int u = 0; u < R; ++u) {
        if (s + u * L < m) {  // conj(p) * q, two independent accumulators
            if (u & 1) {
                d1x = fma(P[u].x, Q[u].x, fma(P[u].y, Q[u].y, d1x));
                d1y = fma(P[u].x, Q[u].y, fma(-P[u].y, Q[u].x, d1y));
            } else {
                d0x = fma(P[u].x, Q[u].x, fma(P[u].y, Q[u].y, d0x));
                d0y = fma(P[u].x, Q[u].y, fma(-P[u].y, Q[u].x, d0y));
            }
        }
    }
    const double2 dot = group_sum2<L>(make_double2(d0x + d1x, d0y + d1y));
    const double mag2 = fma(dot.x, dot.x, dot.y * dot.y);
    if (cp <= drop || cq <= drop || mag2 <= tol2 * cp * cq) return false;
    if (mag2 > 1e-16 * cp * cq) maxrel = 1.0;  // a coupling above 1e-8 relative was rotated
    japply<R>(P, Q, jrot(dot.x, dot.y, cp, cq), cp, cq);
    return true;
}

}  // namespace sslg
