// Host build of paper_2509_20081_b200/csrc/deskew.cuh (tests/test_deskew.py):
// the per-point deskew restatement against the reference's motion_compensate.
// Compiled with -ffp-contract=off so every operation rounds as written.
#include "../../paper_2509_20081_b200/csrc/deskew.cuh"
#include "../../paper_2509_20081_b200/csrc/libm_table.h"

// pts: n x 3 float64 (already downsampled), ts: n times or NULL (linspace)
extern "C" long deskew_host(const dbt_deskew* d, const double* pts, const double* ts, long n, double* out) {
  const double* tab = libm_emu::find_sincostab();
  if (!tab) return -1;
  long rare = 0;
  for (long i = 0; i < n; ++i) {
    const double t = deskew::clip01(ts ? ts[i] : deskew::linspace01(i, n));
    int r = 0;
    deskew::apply(*d, t, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], out + 3 * i, tab, &r);
    rare += r;
  }
  return rare;
}
