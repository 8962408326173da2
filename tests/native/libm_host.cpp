// Host build of paper_2509_20081_b200/csrc/libm_emu.cuh (tests/test_deskew.py):
// the sin/cos restatement against the C library itself. Compiled with
// -ffp-contract=off so every operation rounds exactly as written.
#include "../../paper_2509_20081_b200/csrc/libm_table.h"

extern "C" int libm_tab_found() { return libm_emu::find_sincostab() != nullptr; }
extern "C" int libm_check() {
  const double* t = libm_emu::find_sincostab();
  return t ? libm_emu::check_sincostab(t) : -1;
}
// emulated sin/cos of x[0..n) and the count of results that differ from
// the library's (rare arguments counted as mismatches)
extern "C" long libm_compare(const double* x, long n, double* s_out, double* c_out) {
  const double* t = libm_emu::find_sincostab();
  if (!t) return -1;
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    int rare = 0;
    s_out[i] = libm_emu::sin(x[i], t, &rare);
    c_out[i] = libm_emu::cos(x[i], t, &rare);
    if (rare || libm_emu::bits(s_out[i]) != libm_emu::bits(::sin(x[i])) ||
        libm_emu::bits(c_out[i]) != libm_emu::bits(::cos(x[i])))
      ++bad;
  }
  return bad;
}
