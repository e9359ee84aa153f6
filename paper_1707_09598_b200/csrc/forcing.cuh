// forcing.cuh -- device registry of the closed-form forcings / solutions.
//
// The reference evaluates a Python callable at the physical quadrature
// points (assembly.py:237-245, 290-292); the benchmark configurations use
// the closed forms below (analysis.py:83-167).
#pragma once

#include "../../include/sgiga.h"

namespace sgiga {

template <int D>
__device__ __forceinline__ double forcing_value(int id, const double* x) {
    const double pi = 3.141592653589793;
    switch (id) {
    case SGIGA_FORCING_SIN_PRODUCT: {
        double u = 1.0;
#pragma unroll
        for (int k = 0; k < D; ++k) u *= sin(pi * x[k]);
        return ((double)D * (pi * pi)) * u;
    }
    case SGIGA_FORCING_ANNULUS_POLAR: {
        double xx = x[0], yy = D > 1 ? x[D > 1 ? 1 : 0] : 0.0, s = xx * xx + yy * yy;
        return 32.0 * xx * yy / (s * s) - 24.0 * xx * yy;
    }
    case SGIGA_FORCING_EXP_BUBBLE: {
        double b[D], e = 0.0, tot = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) { b[k] = x[k] * (1.0 - x[k]); e += x[k]; }
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double t = x[m] * (x[m] + 3.0);
#pragma unroll
            for (int k = 0; k < D; ++k) if (k != m) t *= b[k];
            tot += t;
        }
        return exp(e) * tot;
    }
    case SGIGA_FORCING_CUBE_POLY: {
        double b[D], tot = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) b[k] = x[k] * (1.0 - x[k]);
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double t = 1.0;
#pragma unroll
            for (int k = 0; k < D; ++k) if (k != m) t *= b[k];
            tot += 2.0 * t;
        }
        return tot;
    }
    case SGIGA_FORCING_ANNULUS_2D:
    case SGIGA_FORCING_ANNULUS_3D: {
        double xx = x[0], yy = D > 1 ? x[D > 1 ? 1 : 0] : 0.0, x2 = xx * xx, y2 = yy * yy;
        double f2 = 2.0 * xx *
                    (x2 * x2 + 22.0 * x2 * y2 - 5.0 * x2 + 21.0 * y2 * y2 - 45.0 * y2 + 4.0);
        if (id == SGIGA_FORCING_ANNULUS_2D || D < 3) return f2;
        double r2 = x2 + y2, u2 = -(r2 - 1.0) * (r2 - 4.0) * xx * y2;
        return (f2 + pi * pi * u2) * sin(pi * x[D - 1]);
    }
    case SGIGA_FORCING_CONSTANT_ONE: return 1.0;
    default: return 0.0;   // ZERO, LSHAPE (harmonic)
    }
}

// exact solution u and its physical gradient g
template <int D>
__device__ __forceinline__ void solution_value(int id, const double* x, double& u, double* g) {
    const double pi = 3.141592653589793;
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = 0.0;
    u = 0.0;
    switch (id) {
    case SGIGA_FORCING_SIN_PRODUCT: {
        double s[D], c[D];
#pragma unroll
        for (int k = 0; k < D; ++k) { s[k] = sin(pi * x[k]); c[k] = cos(pi * x[k]); }
        u = 1.0;
#pragma unroll
        for (int k = 0; k < D; ++k) u *= s[k];
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double t = pi * c[m];
#pragma unroll
            for (int k = 0; k < D; ++k) if (k != m) t *= s[k];
            g[m] = t;
        }
        return;
    }
    case SGIGA_FORCING_ANNULUS_POLAR: {
        if (D < 2) return;
        double xx = x[0], yy = x[D > 1 ? 1 : 0], s = xx * xx + yy * yy;
        double hh = s - 5.0 + 4.0 / s, hp = 1.0 - 4.0 / (s * s);
        u = 2.0 * xx * yy * hh;
        g[0] = 2.0 * yy * hh + 4.0 * xx * xx * yy * hp;
        g[D > 1 ? 1 : 0] = 2.0 * xx * hh + 4.0 * xx * yy * yy * hp;
        return;
    }
    case SGIGA_FORCING_EXP_BUBBLE: {
        double b[D], e = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) { b[k] = x[k] * (1.0 - x[k]); e += x[k]; }
        e = exp(e);
        u = e;
#pragma unroll
        for (int k = 0; k < D; ++k) u *= b[k];
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double t = e * (b[m] + 1.0 - 2.0 * x[m]);
#pragma unroll
            for (int k = 0; k < D; ++k) if (k != m) t *= b[k];
            g[m] = t;
        }
        return;
    }
    case SGIGA_FORCING_CUBE_POLY: {
        double b[D];
#pragma unroll
        for (int k = 0; k < D; ++k) b[k] = x[k] * (1.0 - x[k]);
        u = 1.0;
#pragma unroll
        for (int k = 0; k < D; ++k) u *= b[k];
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double t = 1.0 - 2.0 * x[m];
#pragma unroll
            for (int k = 0; k < D; ++k) if (k != m) t *= b[k];
            g[m] = t;
        }
        return;
    }
    case SGIGA_FORCING_ANNULUS_2D:
    case SGIGA_FORCING_ANNULUS_3D: {
        if (D < 2) return;
        double xx = x[0], yy = x[D > 1 ? 1 : 0], x2 = xx * xx, y2 = yy * yy, r2 = x2 + y2;
        double u2 = -(r2 - 1.0) * (r2 - 4.0) * xx * y2;
        double gx = -5.0 * x2 * x2 * y2 - 6.0 * x2 * y2 * y2 + 15.0 * x2 * y2 - y2 * y2 * y2 +
                    5.0 * y2 * y2 - 4.0 * y2;
        double gy = -2.0 * x2 * x2 * xx * yy - 8.0 * x2 * xx * y2 * yy + 10.0 * x2 * xx * yy -
                    6.0 * xx * y2 * y2 * yy + 20.0 * xx * y2 * yy - 8.0 * xx * yy;
        if (id == SGIGA_FORCING_ANNULUS_2D || D < 3) {
            u = u2; g[0] = gx; g[D > 1 ? 1 : 0] = gy;
            return;
        }
        double sz = sin(pi * x[D - 1]), cz = cos(pi * x[D - 1]);
        u = u2 * sz;
        g[0] = gx * sz;
        g[1] = gy * sz;
        g[D - 1] = u2 * pi * cz;
        return;
    }
    case SGIGA_FORCING_LSHAPE: {
        if (D < 2) return;
        double xx = x[0], yy = x[D > 1 ? 1 : 0];
        double r = sqrt(xx * xx + yy * yy), th = atan2(yy, xx);
        if (th < 0.0) th += 2.0 * pi;
        if (r == 0.0) return;
        double rr = pow(r, 2.0 / 3.0), s = sin(2.0 * th / 3.0), c = cos(2.0 * th / 3.0);
        double dr = (2.0 / 3.0) * rr / r * s, dth = rr * (2.0 / 3.0) * c;
        u = rr * s;
        g[0] = dr * cos(th) - dth * sin(th) / r;
        g[D > 1 ? 1 : 0] = dr * sin(th) + dth * cos(th) / r;
        return;
    }
    default: return;
    }
}

}  // namespace sgiga
