// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT. CPU FP64 restatement of the
// reference's fixture-generation side, the checker for
// the engine's fixtures.cu. Only tests/, __graft_entry__.smoke() and bench.py's
// CPU legs may load it.
//
// Restated (reference /root/reference/proj/core/src/…):
//   simulator.cpp:14-69    Shepp-Logan ellipsoids, evaluate_ellipsoids, phantom_from_ellipsoids
//   voxelizer.cpp:8-14     grid_for_extent;  voxelizer.cpp:16-37 sample_trilinear
//   simulator.cpp:87-132   box_clip, project_volume (composite-midpoint quadrature)
//   simulator.cpp:134-158  view_rng (splitmix64), add_noise (Poisson + Gaussian, log domain)
//   fdk.cpp:14-134         next_pow2, ramp_response (Ram-Lak / Hann), median_gap, fdk_reconstruct
//   fdk.cpp:136-208        nearest_neighbor_distances (brute force: same minima as the grid search)
//   fdk.cpp:203-247        sample_init_cloud (+ gaussian_cloud.cpp:48-72 add_kernel -> raw)
//   geometry.cpp:76-98,125-138  view_transform, detector_model, pixel_ray
// Eigen::FFT (kissfft backend, un-vendored third-party dependency) is restated as
// a radix-2 complex FFT; only roundoff differs (~1e-15 relative).
// Built with -ffp-contract=off like splatct_oracle.cpp.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

namespace {

struct V3d {
  double v[3];
  double& operator[](int k) { return v[k]; }
  double operator[](int k) const { return v[k]; }
};

struct Grid {
  int dims[3];
  double origin[3], spacing[3];
  double at(const float* vol, int x, int y, int z) const {
    return vol[(static_cast<int64_t>(z) * dims[1] + y) * dims[0] + x];
  }
};
Grid make_grid(const int* dims, const double* origin, const double* spacing) {
  Grid g;
  for (int k = 0; k < 3; ++k) {
    g.dims[k] = dims[k];
    g.origin[k] = origin[k];
    g.spacing[k] = spacing[k];
  }
  return g;
}

// geo = [l_so, l_sd, det_w_mm, det_h_mm, ext_min(3), ext_max(3), near_clip]
struct Scan {
  double l_so, l_sd, dw, dh;
  int w, h, parallel;
};
// res = {W, H, parallel_beam}
Scan make_scan(const double* geo, const int* res) {
  return Scan{geo[0], geo[1], geo[2], geo[3], res[0], res[1], res[2]};
}

struct Rot {
  double m[3][3];
};
// geometry.cpp:76-86
Rot view_rot(double theta) {
  const double s = std::sin(theta), c = std::cos(theta);
  Rot r;
  r.m[0][0] = -s; r.m[0][1] = c; r.m[0][2] = 0.0;
  r.m[1][0] = 0.0; r.m[1][1] = 0.0; r.m[1][2] = -1.0;
  r.m[2][0] = -c; r.m[2][1] = -s; r.m[2][2] = 0.0;
  return r;
}
V3d mul_t(const Rot& r, const V3d& x) {  // r^T x
  V3d o;
  for (int i = 0; i < 3; ++i) o[i] = r.m[0][i] * x[0] + r.m[1][i] * x[1] + r.m[2][i] * x[2];
  return o;
}
V3d mul(const Rot& r, const V3d& x) {
  V3d o;
  for (int i = 0; i < 3; ++i) o[i] = r.m[i][0] * x[0] + r.m[i][1] * x[1] + r.m[i][2] * x[2];
  return o;
}

// geometry.cpp:125-138
void pixel_ray(const Scan& s, double theta, int u, int v, V3d& origin, V3d& dir) {
  const double du = s.dw / s.w, dv = s.dh / s.h;
  const double xd = (u + 0.5) * du - 0.5 * s.dw;
  const double yd = (v + 0.5) * dv - 0.5 * s.dh;
  const Rot r = view_rot(theta);
  if (s.parallel) {  // parallel-beam extension: ray through (xd, yd) along the view axis
    origin = mul_t(r, V3d{{xd, yd, -s.l_so}});
    dir = mul_t(r, V3d{{0.0, 0.0, 1.0}});
    return;
  }
  V3d d{{xd, yd, s.l_sd}};
  const double n = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  for (int k = 0; k < 3; ++k) d[k] = d[k] / n;
  const V3d t{{0.0, 0.0, s.l_so}};
  const V3d src = mul_t(r, t);
  for (int k = 0; k < 3; ++k) origin[k] = -src[k];
  dir = mul_t(r, d);
}

// voxelizer.cpp:16-37
double sample_trilinear(const Grid& g, const float* vol, const V3d& x) {
  int ix[3], f1[3];
  double w[3];
  for (int k = 0; k < 3; ++k) {
    const double gk = (x[k] - g.origin[k]) / g.spacing[k] - 0.5;
    const double c = std::clamp(gk, 0.0, static_cast<double>(g.dims[k] - 1));
    ix[k] = static_cast<int>(std::floor(c));
    ix[k] = std::min(ix[k], g.dims[k] - 1);
    f1[k] = std::min(ix[k] + 1, g.dims[k] - 1);
    w[k] = c - ix[k];
  }
  double out = 0.0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double weight = (dx ? w[0] : 1 - w[0]) * (dy ? w[1] : 1 - w[1]) * (dz ? w[2] : 1 - w[2]);
        out += weight * g.at(vol, dx ? f1[0] : ix[0], dy ? f1[1] : ix[1], dz ? f1[2] : ix[2]);
      }
  return out;
}

// simulator.cpp:90-107
bool box_clip(const V3d& o, const V3d& d, const double* lo, const double* hi, double& t0, double& t1) {
  t0 = 0.0;
  t1 = std::numeric_limits<double>::infinity();
  for (int k = 0; k < 3; ++k) {
    if (std::abs(d[k]) < 1e-15) {
      if (o[k] < lo[k] || o[k] > hi[k]) return false;
      continue;
    }
    double a = (lo[k] - o[k]) / d[k];
    double b = (hi[k] - o[k]) / d[k];
    if (a > b) std::swap(a, b);
    t0 = std::max(t0, a);
    t1 = std::min(t1, b);
  }
  return t1 > t0;
}

// radix-2 FFT (sign -1 forward, +1 inverse without scaling)
void fft(std::vector<std::complex<double>>& a, int sign) {
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = sign * 2.0 * M_PI / static_cast<double>(len);
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < len / 2; ++k) {
        const std::complex<double> w(std::cos(ang * k), std::sin(ang * k));
        const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}

size_t next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

// fdk.cpp:22-43
std::vector<double> ramp_response(size_t padded, double spacing, bool hann) {
  std::vector<std::complex<double>> h(padded, 0.0);
  h[0] = 1.0 / (4.0 * spacing * spacing);
  for (size_t n = 1; n <= padded / 2; ++n)
    if (n % 2 == 1) {
      const double v = -1.0 / (M_PI * M_PI * n * n * spacing * spacing);
      h[n] = v;
      h[padded - n] = v;
    }
  fft(h, -1);
  std::vector<double> r(padded);
  for (size_t k = 0; k < padded; ++k) {
    double x = h[k].real();
    if (hann) x *= 0.5 * (1.0 + std::cos(2.0 * M_PI * static_cast<double>(k) / padded));
    r[k] = x;
  }
  return r;
}

double median_gap(std::vector<double> a) {  // fdk.cpp:45-51
  std::sort(a.begin(), a.end());
  std::vector<double> gaps;
  for (size_t i = 1; i < a.size(); ++i) gaps.push_back(a[i] - a[i - 1]);
  std::sort(gaps.begin(), gaps.end());
  return gaps[gaps.size() / 2];
}

double act_density_inv(double rho) { return rho > 30.0 ? rho : rho + std::log1p(-std::exp(-rho)); }

}  // namespace

extern "C" {

// simulator.cpp:31-69; ell = [n][8] {intensity, a, b, c, x0, y0, z0, phi}
void orc_phantom(int n_ell, const double* ell, const int* dims, const double* lo, const double* hi, float* out) {
  double origin[3], spacing[3], center[3], half[3];
  for (int k = 0; k < 3; ++k) {
    origin[k] = lo[k];
    spacing[k] = (hi[k] - lo[k]) / static_cast<double>(dims[k]);
    center[k] = 0.5 * (lo[k] + hi[k]);
    half[k] = 0.5 * (hi[k] - lo[k]);
  }
#pragma omp parallel for schedule(static)
  for (int z = 0; z < dims[2]; ++z)
    for (int y = 0; y < dims[1]; ++y)
      for (int x = 0; x < dims[0]; ++x) {
        const int idx3[3] = {x, y, z};
        double p[3];
        for (int k = 0; k < 3; ++k) p[k] = (origin[k] + (idx3[k] + 0.5) * spacing[k] - center[k]) / half[k];
        double v = 0.0;
        for (int e = 0; e < n_ell; ++e) {
          const double* E = ell + 8 * e;
          const double dx = p[0] - E[4], dy = p[1] - E[5], dz = p[2] - E[6];
          const double c = std::cos(E[7]), s = std::sin(E[7]);
          const double xr = c * dx + s * dy;
          const double yr = -s * dx + c * dy;
          const double q = (xr * xr) / (E[1] * E[1]) + (yr * yr) / (E[2] * E[2]) + (dz * dz) / (E[3] * E[3]);
          if (q <= 1.0) v += E[0];
        }
        out[(static_cast<int64_t>(z) * dims[1] + y) * dims[0] + x] = static_cast<float>(v);
      }
}

double orc_sample_trilinear(const float* vol, const int* dims, const double* origin, const double* spacing,
                            const double* x) {
  const Grid g = make_grid(dims, origin, spacing);
  return sample_trilinear(g, vol, V3d{{x[0], x[1], x[2]}});
}

// simulator.cpp:109-132 (volume values given as fp32, evaluated in FP64)
int orc_project_volume(const float* vol, const int* dims, const double* origin, const double* spacing,
                       const double* geo, const int* res, double theta, double step_mm, double* out) {
  if (!(step_mm > 0.0)) return 2;
  const Grid g = make_grid(dims, origin, spacing);
  const Scan s = make_scan(geo, res);
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = origin[k];
    hi[k] = origin[k] + spacing[k] * static_cast<double>(dims[k]);
  }
#pragma omp parallel for schedule(static)
  for (int v = 0; v < s.h; ++v)
    for (int u = 0; u < s.w; ++u) {
      V3d o, d;
      pixel_ray(s, theta, u, v, o, d);
      double t0, t1, val = 0.0;
      if (box_clip(o, d, lo, hi, t0, t1)) {
        const int n = std::max(1, static_cast<int>(std::ceil((t1 - t0) / step_mm)));
        const double h = (t1 - t0) / n;
        double sum = 0.0;
        for (int i = 0; i < n; ++i) {
          V3d x;
          for (int k = 0; k < 3; ++k) x[k] = o[k] + (t0 + (i + 0.5) * h) * d[k];
          sum += sample_trilinear(g, vol, x);
        }
        val = sum * h;
      }
      out[static_cast<int64_t>(v) * s.w + u] = val;
    }
  return 0;
}

// simulator.cpp:134-141
uint64_t orc_view_seed(uint64_t master, int view) {
  uint64_t z = master + 0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(view) + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// simulator.cpp:143-157 on one view (clean log image given as fp32)
int orc_add_noise(const float* clean, int n, double i0, double gauss_sigma, uint64_t seed, int view, double* out) {
  if (!(i0 > 0.0)) return 2;
  std::mt19937_64 rng(orc_view_seed(seed, view));
  std::normal_distribution<double> gauss(0.0, 1.0);
  const double log_i0 = std::log(i0);
  for (int i = 0; i < n; ++i) {
    const double lambda = i0 * std::exp(-static_cast<double>(clean[i]));
    std::poisson_distribution<long> poisson(lambda);
    double counts = static_cast<double>(poisson(rng));
    if (gauss_sigma > 0.0) counts += gauss_sigma * gauss(rng);
    counts = std::max(counts, 1.0);
    out[i] = log_i0 - std::log(counts);
  }
  return 0;
}

// fdk.cpp:53-134. images [n][h][w] fp32; window 0 ramp, 1 hann, 2 auto (hann when n < 100).
int orc_fdk(const float* images, int n_views, const double* geo, const int* res, const double* angles,
            const int* dims, const double* origin, const double* spacing, int window, double* out) {
  if (n_views < 2) return 3;
  const Scan s = make_scan(geo, res);
  const int w = s.w, h = s.h;
  const double du = s.dw / w, dv = s.dh / h;
  const double mag = s.l_so / s.l_sd;
  const double da = du * mag;
  const bool hann = window == 1 || (window == 2 && n_views < 100);
  const size_t padded = next_pow2(static_cast<size_t>(2 * w));
  const std::vector<double> resp = ramp_response(padded, da, hann);
  std::vector<double> filt(static_cast<size_t>(n_views) * w * h);
#pragma omp parallel for schedule(static)
  for (int view = 0; view < n_views; ++view) {
    std::vector<std::complex<double>> row(padded);
    for (int v = 0; v < h; ++v) {
      const double yd = (v + 0.5) * dv - 0.5 * s.dh;
      for (size_t u = 0; u < padded; ++u) row[u] = 0.0;
      for (int u = 0; u < w; ++u) {
        const double xd = (u + 0.5) * du - 0.5 * s.dw;
        const double cosw = s.l_sd / std::sqrt(s.l_sd * s.l_sd + xd * xd + yd * yd);
        row[u] = static_cast<double>(images[(static_cast<size_t>(view) * h + v) * w + u]) * cosw;
      }
      fft(row, -1);
      for (size_t k = 0; k < padded; ++k) row[k] *= resp[k];
      fft(row, +1);
      for (int u = 0; u < w; ++u)
        filt[(static_cast<size_t>(view) * h + v) * w + u] = row[u].real() / static_cast<double>(padded) * da;
    }
  }
  const double dtheta = median_gap(std::vector<double>(angles, angles + n_views));
  std::vector<Rot> rots(n_views);
  for (int i = 0; i < n_views; ++i) rots[i] = view_rot(angles[i]);
  const int nx = dims[0], ny = dims[1], nz = dims[2];
#pragma omp parallel for schedule(static)
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const V3d p{{origin[0] + (x + 0.5) * spacing[0], origin[1] + (y + 0.5) * spacing[1],
                     origin[2] + (z + 0.5) * spacing[2]}};
        double acc = 0.0;
        for (int i = 0; i < n_views; ++i) {
          V3d pc = mul(rots[i], p);
          pc[2] += s.l_so;
          if (pc[2] <= 0.0) continue;
          const double xd = pc[0] * s.l_sd / pc[2];
          const double yd = pc[1] * s.l_sd / pc[2];
          const double uc = (xd + 0.5 * s.dw) / du - 0.5;
          const double vc = (yd + 0.5 * s.dh) / dv - 0.5;
          if (uc < 0.0 || uc > w - 1 || vc < 0.0 || vc > h - 1) continue;
          const int u0 = std::min(static_cast<int>(uc), w - 2);
          const int v0 = std::min(static_cast<int>(vc), h - 2);
          const double fu = uc - u0, fv = vc - v0;
          const double* q = filt.data() + static_cast<size_t>(i) * w * h;
          const double val = (1 - fu) * (1 - fv) * q[v0 * w + u0] + fu * (1 - fv) * q[v0 * w + u0 + 1] +
                             (1 - fu) * fv * q[(v0 + 1) * w + u0] + fu * fv * q[(v0 + 1) * w + u0 + 1];
          const double ratio = s.l_so / pc[2];
          acc += ratio * ratio * val;
        }
        out[(static_cast<int64_t>(z) * ny + y) * nx + x] = 0.5 * dtheta * acc;
      }
  return 0;
}

// fdk.cpp:136-201 (the grid search returns the brute-force minima)
void orc_nn_distances(int n, const double* pts, double* out) {
  if (n < 2) {
    for (int i = 0; i < n; ++i) out[i] = 0.0;
    return;
  }
#pragma omp parallel for schedule(dynamic, 64)
  for (int i = 0; i < n; ++i) {
    double best = std::numeric_limits<double>::infinity();
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = pts[3 * i] - pts[3 * j], dy = pts[3 * i + 1] - pts[3 * j + 1],
                   dz = pts[3 * i + 2] - pts[3 * j + 2];
      best = std::min(best, dx * dx + dy * dy + dz * dz);
    }
    out[i] = std::sqrt(best);
  }
}

// fdk.cpp:203-247: returns 3 (TooFewOccupiedVoxels) when too few voxels pass.
// outputs raw arrays (gaussian_cloud.cpp:48-72 add_kernel): rho_raw[count],
// pos[3count], scale_raw[3count], rot[4count]
int orc_sample_init_cloud(void* rp, const float* vol, const int* dims, const double* origin, const double* spacing,
                          int count, double threshold, double density_scale, double s_min, double* rho_raw,
                          double* pos, double* scale_raw, double* rot) {
  auto& rng = *static_cast<std::mt19937_64*>(rp);
  const Grid g = make_grid(dims, origin, spacing);
  const int64_t nvox = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
  std::vector<int64_t> occ;
  for (int64_t i = 0; i < nvox; ++i)
    if (static_cast<double>(vol[i]) > threshold) occ.push_back(i);
  if (static_cast<int64_t>(occ.size()) < count) return 3;
  for (int i = 0; i < count; ++i) {
    std::uniform_int_distribution<size_t> pick(i, occ.size() - 1);
    std::swap(occ[i], occ[pick(rng)]);
  }
  std::uniform_real_distribution<double> jitter(-0.5, 0.5);
  for (int i = 0; i < count; ++i) {
    const int64_t idx = occ[i];
    const int x = static_cast<int>(idx % dims[0]);
    const int y = static_cast<int>((idx / dims[0]) % dims[1]);
    const int z = static_cast<int>(idx / (static_cast<int64_t>(dims[0]) * dims[1]));
    const int xyz[3] = {x, y, z};
    for (int k = 0; k < 3; ++k) {
      double p = origin[k] + (xyz[k] + 0.5) * spacing[k];
      p += jitter(rng) * spacing[k];
      pos[3 * i + k] = p;
    }
  }
  std::vector<double> nn(count);
  orc_nn_distances(count, pos, nn.data());
  for (int i = 0; i < count; ++i) {
    const double s = std::max(nn[i], s_min * (1.0 + 1e-6));
    const double rho = std::max(density_scale * sample_trilinear(g, vol, V3d{{pos[3 * i], pos[3 * i + 1],
                                                                               pos[3 * i + 2]}}), 1e-6);
    rho_raw[i] = act_density_inv(rho);
    for (int k = 0; k < 3; ++k) scale_raw[3 * i + k] = std::log(s - s_min);
    rot[4 * i] = 1.0;
    rot[4 * i + 1] = rot[4 * i + 2] = rot[4 * i + 3] = 0.0;
  }
  return 0;
}

}  // extern "C"
