// Host-side random streams of the reference trainer (product host code, not
// the oracle): trainer.cpp:254-258 seeds ONE std::mt19937_64 with cfg.seed and
// draws from it, in iteration order,
//   * std::shuffle of the view order at every epoch start (trainer.cpp:269-273;
//     the order is reshuffled in place, not reset),
//   * random_subvolume_spec's three uniform(0,1) draws (voxelizer.cpp:226-239),
//   * adaptive_control's split draws: one std::normal_distribution(0,1) object
//     per call, 3 draws per child in the order z, y, x (GCC evaluates the
//     Vec3(gauss*s.x, gauss*s.y, gauss*s.z) arguments right to left;
//     trainer.cpp:184,213-216).
// The same libstdc++ engine and distributions as the reference build, so the
// engine's train loop consumes an identical stream (seed parity).
#include <algorithm>
#include <cstdint>
#include <new>
#include <random>

#include "sct_internal.cuh"

struct sct_rng {
  std::mt19937_64 eng;
};

extern "C" {

int sct_rng_create(uint64_t seed, sct_rng** out) {
  if (!out) {
    sct::set_error("ConfigError: null output handle");
    return SCT_ERR_CONFIG;
  }
  *out = new (std::nothrow) sct_rng{std::mt19937_64(seed)};
  if (!*out) {
    sct::set_error("host allocation failed");
    return SCT_ERR_OTHER;
  }
  return SCT_OK;
}

int sct_rng_destroy(sct_rng* r) {
  delete r;
  return SCT_OK;
}

int sct_rng_shuffle(sct_rng* r, int32_t* values, int32_t n) {
  if (!r || (n > 0 && !values)) {
    sct::set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  std::shuffle(values, values + n, r->eng);
  return SCT_OK;
}

int sct_rng_subvolume_origin(sct_rng* r, const double lo[3], const double hi[3], const double spacing[3], int32_t d,
                             double origin[3]) {
  if (!r || !lo || !hi || !spacing || !origin) {
    sct::set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int k = 0; k < 3; ++k) {
    const double span = (hi[k] - lo[k]) - d * spacing[k];
    const double u = uni(r->eng);
    origin[k] = span > 0.0 ? lo[k] + u * span : 0.5 * (lo[k] + hi[k]) - 0.5 * d * spacing[k];
  }
  return SCT_OK;
}

int sct_rng_normal(sct_rng* r, int64_t n, double* out) {
  if (!r || (n > 0 && !out)) {
    sct::set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int64_t i = 0; i < n; ++i) out[i] = gauss(r->eng);
  return SCT_OK;
}

int sct_rng_uniform(sct_rng* r, int64_t n, double lo, double hi, double* out) {
  if (!r || (n > 0 && !out)) {
    sct::set_error("ConfigError: null argument");
    return SCT_ERR_CONFIG;
  }
  std::uniform_real_distribution<double> uni(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = uni(r->eng);
  return SCT_OK;
}

}  // extern "C"
