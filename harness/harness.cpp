// Seeded synthetic-input generators for the TV-reconstruction hot path.
//
// This module produces INPUTS only: the Siddon system matrix A (CSR of ray/voxel
// intersection lengths), the ellipsoid phantom x_true, the simulated data
// b = A x_true + e (§IV-A "Simulation setup", Eq. (11)), and
// seeded uniform/Gaussian streams.  It contains none of the method's arithmetic
// (no objective, TV, gradient, projection or solver step).  Both the oracle
// (oracle/) and the CUDA path (paper_1105_4002_b200/) consume its outputs; it
// imports neither.
//
// Conventions follow SURVEY.md §8(c): C4 (layouts), C15 (Siddon), C16 (noise),
// C17 (phantom, SplitMix64 + Box-Muller).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---------------------------------------------------------------- RNG (C17)
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  // 53-bit uniform in [0,1)
  double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// ------------------------------------------------------------- Siddon (C15)
// Segment list of one ray p(t) = p0 + t d through an nx x ny (x nz) unit-voxel
// box centred at the origin; voxel i on an axis of n voxels spans
// [i - n/2, i - n/2 + 1).  Crossings with every axis-normal grid plane are
// collected, sorted and uniqued; each consecutive pair is a segment of length
// dt (|d| = 1), owned by the voxel containing its midpoint (floor rule);
// segments of length <= 1e-9 and segments outside the box are dropped.
constexpr double kDropLen = 1e-9;

struct Seg {
  int64_t col;
  double len;
};

void trace_ray(const double p0[3], const double d[3], const int n[3], int ndim,
               std::vector<double>& ts, std::vector<Seg>& out) {
  ts.clear();
  out.clear();
  for (int a = 0; a < ndim; ++a) {
    if (d[a] == 0.0) continue;
    const double h = 0.5 * n[a];
    for (int i = 0; i <= n[a]; ++i) {
      const double plane = (double)i - h;
      ts.push_back((plane - p0[a]) / d[a]);
    }
  }
  if (ts.size() < 2) return;
  std::sort(ts.begin(), ts.end());
  ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
  for (size_t k = 0; k + 1 < ts.size(); ++k) {
    const double len = ts[k + 1] - ts[k];
    if (len <= kDropLen) continue;
    const double tm = 0.5 * (ts[k] + ts[k + 1]);
    int64_t idx[3] = {0, 0, 0};
    bool inside = true;
    for (int a = 0; a < ndim; ++a) {
      const double p = p0[a] + tm * d[a];
      const double f = std::floor(p + 0.5 * n[a]);
      if (f < 0.0 || f >= (double)n[a]) { inside = false; break; }
      idx[a] = (int64_t)f;
    }
    if (!inside) continue;
    int64_t col = (ndim == 3) ? ((idx[2] * n[1] + idx[1]) * n[0] + idx[0])
                              : (idx[1] * n[0] + idx[0]);
    out.push_back({col, len});
  }
  std::sort(out.begin(), out.end(), [](const Seg& a, const Seg& b) { return a.col < b.col; });
}

// View direction for angle index v of V over [0, 180deg): exact at 0 and 90 deg.
void view_dir(int v, int V, double* c, double* s) {
  if (v == 0) { *c = 1.0; *s = 0.0; return; }
  if (2 * v == V) { *c = 0.0; *s = 1.0; return; }
  const double th = M_PI * (double)v / (double)V;
  *c = std::cos(th);
  *s = std::sin(th);
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- 2D slice
// One axial slice's system matrix, rows i = v*nb + b (view-major within the
// slice, C4), columns iy*nx + ix.  Call with col/val == NULL to obtain the row
// pointer and nnz; then again with buffers of size nnz.  Returns nnz.
int64_t hx_siddon2d(int nx, int ny, int V, int nb, int64_t* row_ptr, int32_t* col,
                    float* val) {
  const int n[3] = {nx, ny, 1};
  const int64_t m = (int64_t)V * nb;
  std::vector<int64_t> cnt(m, 0);
  std::vector<std::vector<Seg>> segs_per_thread;
#pragma omp parallel
  {
    std::vector<double> ts;
    std::vector<Seg> segs;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      const int v = (int)(i / nb), b = (int)(i % nb);
      double c, s;
      view_dir(v, V, &c, &s);
      const double d[3] = {c, s, 0.0};
      const double u[2] = {-s, c};
      const double sb = (double)b - 0.5 * (double)(nb - 1);
      const double p0[3] = {sb * u[0], sb * u[1], 0.0};
      trace_ray(p0, d, n, 2, ts, segs);
      cnt[i] = (int64_t)segs.size();
      if (col && val) {
        int64_t off = row_ptr[i];
        for (size_t k = 0; k < segs.size(); ++k) {
          col[off + k] = (int32_t)segs[k].col;
          val[off + k] = (float)segs[k].len;  // fp64 length rounded to fp32 (RN)
        }
      }
    }
  }
  if (!(col && val)) {
    row_ptr[0] = 0;
    for (int64_t i = 0; i < m; ++i) row_ptr[i + 1] = row_ptr[i] + cnt[i];
  }
  return row_ptr[m];
}

// Replicate one slice matrix over nz slices: slice-major rows
// i = (z*V + v)*nb + b and columns offset by z*nx*ny (C4).  A is
// block-diagonal by slice.
void hx_replicate_slices(int64_t m_s, int64_t nnz_s, const int64_t* rp_s, const int32_t* col_s,
                         const float* val_s, int64_t slice_cols, int nz, int64_t* row_ptr,
                         int32_t* col, float* val) {
#pragma omp parallel for schedule(static)
  for (int z = 0; z < nz; ++z) {
    const int64_t r0 = (int64_t)z * m_s, e0 = (int64_t)z * nnz_s;
    const int32_t coff = (int32_t)((int64_t)z * slice_cols);
    for (int64_t i = 0; i < m_s; ++i) row_ptr[r0 + i] = e0 + rp_s[i];
    for (int64_t k = 0; k < nnz_s; ++k) {
      col[e0 + k] = col_s[k] + coff;
      val[e0 + k] = val_s[k];
    }
  }
  row_ptr[(int64_t)nz * m_s] = (int64_t)nz * nnz_s;
}

// ---------------------------------------------------------- 3D tilted (c5)
// Non-separable parallel beam: V views, detector R x C pixels.  For view v,
// theta_v = 180deg*v/V, tilt phi_v = phimax*(2v/(V-1) - 1);
// d = (cos phi cos th, cos phi sin th, sin phi), u = (-sin th, cos th, 0),
// w = d x u; pixel (r, c) centre (c-(C-1)/2) u + (r-(R-1)/2) w.  Rows are
// view-major i = (v*R + r)*C + c (C4).  Columns (iz*ny + iy)*nx + ix.
int64_t hx_siddon3d_views(int nx, int ny, int nz, int V, int R, int C, double phimax_deg,
                          int v0, int v1, int64_t* row_ptr, int32_t* col, float* val);
int64_t hx_siddon3d(int nx, int ny, int nz, int V, int R, int C, double phimax_deg,
                    int64_t* row_ptr, int32_t* col, float* val) {
  return hx_siddon3d_views(nx, ny, nz, V, R, C, phimax_deg, 0, V, row_ptr, col, val);
}

// The rows of views [v0, v1) only (a contiguous block of the view-major rows, for one rank of a
// view-sharded run): row_ptr has (v1 - v0) R C + 1 entries starting at 0; the rays are those of
// the full geometry (the tilt and angle of view v depend on V, not on the block).
int64_t hx_siddon3d_views(int nx, int ny, int nz, int V, int R, int C, double phimax_deg,
                          int v0, int v1, int64_t* row_ptr, int32_t* col, float* val) {
  const int n[3] = {nx, ny, nz};
  const int64_t m = (int64_t)(v1 - v0) * R * C;
  const int64_t i0 = (int64_t)v0 * R * C;
  std::vector<int64_t> cnt(col && val ? 0 : m, 0);
#pragma omp parallel
  {
    std::vector<double> ts;
    std::vector<Seg> segs;
#pragma omp for schedule(dynamic, 64)
    for (int64_t il = 0; il < m; ++il) {
      const int64_t i = i0 + il;
      const int v = (int)(i / ((int64_t)R * C));
      const int r = (int)((i / C) % R), cc = (int)(i % C);
      double ct, st;
      view_dir(v, V, &ct, &st);
      const double phi = (V > 1 ? phimax_deg * (2.0 * v / (double)(V - 1) - 1.0) : 0.0) * M_PI / 180.0;
      const double cp = std::cos(phi), sp = std::sin(phi);
      const double d[3] = {cp * ct, cp * st, sp};
      const double u[3] = {-st, ct, 0.0};
      const double w[3] = {d[1] * u[2] - d[2] * u[1], d[2] * u[0] - d[0] * u[2],
                           d[0] * u[1] - d[1] * u[0]};
      const double a = (double)cc - 0.5 * (C - 1), bb = (double)r - 0.5 * (R - 1);
      const double p0[3] = {a * u[0] + bb * w[0], a * u[1] + bb * w[1], a * u[2] + bb * w[2]};
      trace_ray(p0, d, n, 3, ts, segs);
      if (col && val) {
        int64_t off = row_ptr[il];
        for (size_t k = 0; k < segs.size(); ++k) {
          col[off + k] = (int32_t)segs[k].col;
          val[off + k] = (float)segs[k].len;
        }
      } else {
        cnt[il] = (int64_t)segs.size();
      }
    }
  }
  if (!(col && val)) {
    row_ptr[0] = 0;
    for (int64_t i = 0; i < m; ++i) row_ptr[i + 1] = row_ptr[i] + cnt[i];
  }
  return row_ptr[m];
}

// 3D parallel beam with view directions spread over the unit sphere (the paper's own
// geometry).  Reading: golden-spiral directions on the half sphere (d and -d
// give the same parallel projection): cos(theta_v) = 1 - (v + 1/2)/V, azimuth v * pi (3 - sqrt 5).
// Detector R x C of unit pixels centred on the origin, spanned by u = (a x d)/|a x d| (a = e_z,
// or e_x when d is within ~26 deg of e_z) and w = d x u.  Rows view-major: (v R + r) C + c.
int64_t hx_siddon_sphere(int nx, int ny, int nz, int V, int R, int C, int64_t* row_ptr,
                         int32_t* col, float* val) {
  const int n[3] = {nx, ny, nz};
  const int64_t m = (int64_t)V * R * C;
  std::vector<int64_t> cnt(col && val ? 0 : m, 0);
  const double golden = M_PI * (3.0 - std::sqrt(5.0));
#pragma omp parallel
  {
    std::vector<double> ts;
    std::vector<Seg> segs;
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < m; ++i) {
      const int v = (int)(i / ((int64_t)R * C));
      const int r = (int)((i / C) % R), cc = (int)(i % C);
      const double ct = 1.0 - (v + 0.5) / (double)V, st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
      const double ph = golden * v;
      const double d[3] = {st * std::cos(ph), st * std::sin(ph), ct};
      const double a[3] = {std::fabs(ct) < 0.9 ? 0.0 : 1.0, 0.0, std::fabs(ct) < 0.9 ? 1.0 : 0.0};
      double u[3] = {a[1] * d[2] - a[2] * d[1], a[2] * d[0] - a[0] * d[2], a[0] * d[1] - a[1] * d[0]};
      const double un = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
      for (double& q : u) q /= un;
      const double w[3] = {d[1] * u[2] - d[2] * u[1], d[2] * u[0] - d[0] * u[2],
                           d[0] * u[1] - d[1] * u[0]};
      const double pa = (double)cc - 0.5 * (C - 1), pb = (double)r - 0.5 * (R - 1);
      const double p0[3] = {pa * u[0] + pb * w[0], pa * u[1] + pb * w[1], pa * u[2] + pb * w[2]};
      trace_ray(p0, d, n, 3, ts, segs);
      if (col && val) {
        int64_t off = row_ptr[i];
        for (size_t k = 0; k < segs.size(); ++k) {
          col[off + k] = (int32_t)segs[k].col;
          val[off + k] = (float)segs[k].len;
        }
      } else {
        cnt[i] = (int64_t)segs.size();
      }
    }
  }
  if (!(col && val)) {
    row_ptr[0] = 0;
    for (int64_t i = 0; i < m; ++i) row_ptr[i + 1] = row_ptr[i] + cnt[i];
  }
  return row_ptr[m];
}

// Simulated projections y = A x (fp64 accumulation of fp32 entries): the
// "forward mapping of the discretized image" of the simulation setup
// (Eq. (11)).  Data generation only.
void hx_simulate_projections(int64_t m, const int64_t* row_ptr, const int32_t* col,
                             const float* val, const float* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += (double)val[k] * (double)x[col[k]];
    y[i] = s;
  }
}

// --------------------------------------------------------- phantom (C17)
// n_ell additive ellipsoids in normalised voxel-centre coordinates [-1,1]^3.
// Per ellipsoid, draws in order: centre (3 x U[-0.5,0.5]), semi-axes
// (3 x U[0.1,0.45]), ZYX Euler angles (3 x U[0,2pi)), value U[0.2,1.0].
// The sum is clipped to [0,1] and stored as fp32.
void hx_phantom(int nx, int ny, int nz, int n_ell, uint64_t seed, float* out) {
  struct Ell { double c[3], a[3], R[9], val; };
  std::vector<Ell> E(n_ell);
  SplitMix64 rng(seed);
  for (int e = 0; e < n_ell; ++e) {
    Ell& q = E[e];
    for (int k = 0; k < 3; ++k) q.c[k] = -0.5 + rng.uniform();
    for (int k = 0; k < 3; ++k) q.a[k] = 0.1 + 0.35 * rng.uniform();
    double ang[3];
    for (int k = 0; k < 3; ++k) ang[k] = 2.0 * M_PI * rng.uniform();
    q.val = 0.2 + 0.8 * rng.uniform();
    const double cz = std::cos(ang[0]), sz = std::sin(ang[0]);
    const double cy = std::cos(ang[1]), sy = std::sin(ang[1]);
    const double cx = std::cos(ang[2]), sx = std::sin(ang[2]);
    // R = Rz * Ry * Rx
    const double Rm[9] = {cz * cy, cz * sy * sx - sz * cx, cz * sy * cx + sz * sx,
                          sz * cy, sz * sy * sx + cz * cx, sz * sy * cx - cz * sx,
                          -sy,     cy * sx,                cy * cx};
    std::memcpy(q.R, Rm, sizeof(Rm));
  }
#pragma omp parallel for schedule(static)
  for (int iz = 0; iz < nz; ++iz) {
    const double pz = ((double)iz - 0.5 * nz + 0.5) / (0.5 * nz);
    for (int iy = 0; iy < ny; ++iy) {
      const double py = ((double)iy - 0.5 * ny + 0.5) / (0.5 * ny);
      for (int ix = 0; ix < nx; ++ix) {
        const double px = ((double)ix - 0.5 * nx + 0.5) / (0.5 * nx);
        double s = 0.0;
        for (const Ell& q : E) {
          const double dx = px - q.c[0], dy = py - q.c[1], dz = pz - q.c[2];
          // body coordinates = R^T (p - c)
          const double bx = q.R[0] * dx + q.R[3] * dy + q.R[6] * dz;
          const double by = q.R[1] * dx + q.R[4] * dy + q.R[7] * dz;
          const double bz = q.R[2] * dx + q.R[5] * dy + q.R[8] * dz;
          const double r2 = (bx / q.a[0]) * (bx / q.a[0]) + (by / q.a[1]) * (by / q.a[1]) +
                            (bz / q.a[2]) * (bz / q.a[2]);
          if (r2 <= 1.0) s += q.val;
        }
        s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
        out[((int64_t)iz * ny + iy) * nx + ix] = (float)s;
      }
    }
  }
}

// ------------------------------------------------------ seeded streams (C17)
void hx_uniform(int64_t n, uint64_t seed, double* out) {
  SplitMix64 rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.uniform();
}

// Box-Muller: each pair of uniforms (u1, u2) yields two normals
// sqrt(-2 ln(1-u1)) * (cos 2pi u2, sin 2pi u2).
void hx_normal(int64_t n, uint64_t seed, double* out) {
  SplitMix64 rng(seed);
  for (int64_t i = 0; i < n; i += 2) {
    const double u1 = rng.uniform(), u2 = rng.uniform();
    const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
    out[i] = rad * std::cos(2.0 * M_PI * u2);
    if (i + 1 < n) out[i + 1] = rad * std::sin(2.0 * M_PI * u2);
  }
}

}  // extern "C"
