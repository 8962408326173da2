// Host build of paper_2509_20081_b200/csrc/svml_emu.cuh for validating the
// SVML restatement against numpy on CPU (tests/test_svml_emu.py). Compiled
// with -ffp-contract=off so every operation rounds exactly as written.
#include "../../paper_2509_20081_b200/csrc/svml_emu.cuh"

extern "C" void svml_atan2_arr(const double* y, const double* x, long n, const uint16_t* tab, double* out, int* rare) {
  for (long i = 0; i < n; ++i) out[i] = svml::atan2(y[i], x[i], tab, rare + i);
}
extern "C" void svml_asin_arr(const double* x, long n, const uint16_t* tab, double* out) {
  for (long i = 0; i < n; ++i) out[i] = svml::asin(x[i], tab);
}
