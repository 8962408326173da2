// libm_table.h — host-side access to the C library's sin/cos table for the
// libm_emu.cuh restatement (see there): the table is located in the loaded
// libm image at run time (never copied into this repository) and the
// restatement is checked against the library's own sin/cos before use.
#pragma once

#include <dlfcn.h>
#include <link.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "libm_emu.cuh"

namespace libm_emu {

struct TabSearch {
  const double* found = nullptr;
};

// The table starts with sin/cos of 0 and of 1/128: 0, 0, 1, 0, sin(1/128)
// (correctly rounded), its low part, cos(1/128), its low part.
inline int tab_scan(struct dl_phdr_info* info, size_t, void* data) {
  TabSearch* ts = static_cast<TabSearch*>(data);
  if (ts->found || !info->dlpi_name || !strstr(info->dlpi_name, "libm.so")) return 0;
  const double sn1 = 0x1.fffeaaaaeeeefp-8, cs1 = 0x1.fffc000155552p-1;
  for (int i = 0; i < info->dlpi_phnum; ++i) {
    const ElfW(Phdr)& ph = info->dlpi_phdr[i];
    if (ph.p_type != PT_LOAD || (ph.p_flags & PF_W)) continue;
    const unsigned char* base = reinterpret_cast<const unsigned char*>(info->dlpi_addr + ph.p_vaddr);
    const size_t n = ph.p_memsz / 8;
    const double* d = reinterpret_cast<const double*>(base);  // segments are page aligned
    for (size_t k = 0; k + kTabEntries <= n; ++k) {
      if (d[k + 4] != sn1 || d[k + 6] != cs1) continue;
      if (d[k] != 0.0 || d[k + 1] != 0.0 || d[k + 2] != 1.0 || d[k + 3] != 0.0) continue;
      ts->found = d + k;
      return 1;
    }
  }
  return 0;
}

// The table inside the process's libm, or nullptr.
inline const double* find_sincostab() {
  void* h = dlopen("libm.so.6", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libm.so.6", RTLD_NOW);
  if (!h) return nullptr;
  TabSearch ts;
  dl_iterate_phdr(tab_scan, &ts);
  return ts.found;
}

// The restatement against the library on arguments covering every branch
// (both signs, each range, table boundaries, the reduction). Returns the
// number of mismatching results (0: the device may use it).
inline int check_sincostab(const double* tab) {
  typedef double (*Fn)(double);
  void* h = dlopen("libm.so.6", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libm.so.6", RTLD_NOW);
  if (!h) return -1;
  Fn lsin = reinterpret_cast<Fn>(dlsym(h, "sin")), lcos = reinterpret_cast<Fn>(dlsym(h, "cos"));
  if (!lsin || !lcos) return -1;
  int bad = 0;
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < 200000; ++i) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    const double u = (double)(s >> 11) * 0x1p-53;  // [0, 1)
    double x;
    switch (i % 5) {
      case 0: x = u * 0.13; break;                 // Taylor range
      case 1: x = u * 0.86; break;                 // table range
      case 2: x = 0.85 + u * 1.6; break;           // pi/2 - |x|
      case 3: x = 2.4 + u * 8.0; break;            // reduction
      default: x = ldexp(u, -(int)(s & 31)); break;  // small magnitudes
    }
    if (s & (1ull << 40)) x = -x;
    int rare = 0;
    const double a = sin(x, tab, &rare), b = cos(x, tab, &rare);
    if (rare || bits(a) != bits(lsin(x)) || bits(b) != bits(lcos(x))) ++bad;
  }
  return bad;
}

}  // namespace libm_emu
