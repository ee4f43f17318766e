// OBJ frame export, host C++.
//
// Replaces export_frame / surface_subset (intact/io_utils.py:22-43): only
// the vertices the triangles reference are written, in ascending id order,
// and faces are renumbered against them (1-based).  Coordinates are written
// as Python's repr(float): the shortest digit string that round-trips
// (std::to_chars), laid out by Python's rules — positional notation when
// the decimal exponent is in [-4, 16), scientific with a signed, at least
// two-digit exponent otherwise, ".0" on integral values.  The file is
// byte-identical to the reference's.  Lines are formatted in parallel
// chunks and written in order.

#include <charconv>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ibf.h"

namespace ibf {
void set_error(const std::string& msg);
}

namespace {

// Python repr of a finite or non-finite double
void put_repr(std::string& out, double v) {
  if (std::isnan(v)) {
    out += "nan";
    return;
  }
  if (std::isinf(v)) {
    out += v < 0 ? "-inf" : "inf";
    return;
  }
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  *r.ptr = '\0';
  // buf = [-]d[.ddd]e(+|-)xx
  const char* p = buf;
  if (*p == '-') {
    out += '-';
    ++p;
  }
  char digits[32];
  int nd = 0;
  const char* e = std::strchr(p, 'e');
  for (const char* q = p; q < e; ++q)
    if (*q != '.') digits[nd++] = *q;
  const int exp10 = std::atoi(e + 1);
  if (nd == 1 && digits[0] == '0') {
    out += "0.0";
    return;
  }
  const int decpt = exp10 + 1;  // value = 0.d1d2... * 10^decpt
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) {
      out += "0.";
      out.append(-decpt, '0');
      out.append(digits, nd);
    } else if (decpt < nd) {
      out.append(digits, decpt);
      out += '.';
      out.append(digits + decpt, nd - decpt);
    } else {
      out.append(digits, nd);
      out.append(decpt - nd, '0');
      out += ".0";
    }
  } else {
    out += digits[0];
    if (nd > 1) {
      out += '.';
      out.append(digits + 1, nd - 1);
    }
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
    out += eb;
  }
}

void put_int(std::string& out, long long v) {
  char buf[24];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  out.append(buf, r.ptr - buf);
}

template <class F>
void parallel_chunks(int64_t n, int threads, std::vector<std::string>& parts, F fmt) {
  const int64_t per = (n + threads - 1) / threads;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const int64_t a = t * per, b = std::min<int64_t>(n, a + per);
    if (a >= b) break;
    pool.emplace_back([&, t, a, b] { fmt(parts[t], a, b); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" int ibf_export_obj(const char* path, const double* positions, int64_t n_positions, const int64_t* tris,
                              int64_t n_tris, int n_threads) {
  if (!path || n_positions < 0 || n_tris < 0 || (n_tris && !tris) || (n_positions && !positions)) {
    ibf::set_error("ibf_export_obj: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  // used = unique(triangles), remap[used] = 0..len(used)-1
  int64_t top = -1;
  for (int64_t k = 0; k < 3 * n_tris; ++k) {
    if (tris[k] < 0 || tris[k] >= n_positions) {
      ibf::set_error("ibf_export_obj: triangle index " + std::to_string(tris[k]) + " out of range");
      return IBF_ERR_BAD_ARG;
    }
    top = std::max<int64_t>(top, tris[k]);
  }
  std::vector<int64_t> remap(top + 1, -1);
  for (int64_t k = 0; k < 3 * n_tris; ++k) remap[tris[k]] = 0;
  std::vector<int64_t> used;
  for (int64_t v = 0; v <= top; ++v)
    if (remap[v] == 0) {
      remap[v] = (int64_t)used.size();
      used.push_back(v);
    }
  const int64_t nv = (int64_t)used.size();
  int threads = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  threads = std::max(1, std::min(threads, 256));
  std::vector<std::string> vparts(threads), fparts(threads);
  parallel_chunks(nv, threads, vparts, [&](std::string& s, int64_t a, int64_t b) {
    s.reserve((size_t)(b - a) * 64);
    for (int64_t i = a; i < b; ++i) {
      const double* p = positions + 3 * used[i];
      s += "v ";
      put_repr(s, p[0]);
      s += ' ';
      put_repr(s, p[1]);
      s += ' ';
      put_repr(s, p[2]);
      s += '\n';
    }
  });
  parallel_chunks(n_tris, threads, fparts, [&](std::string& s, int64_t a, int64_t b) {
    s.reserve((size_t)(b - a) * 24);
    for (int64_t t = a; t < b; ++t) {
      s += "f ";
      put_int(s, remap[tris[3 * t]] + 1);
      s += ' ';
      put_int(s, remap[tris[3 * t + 1]] + 1);
      s += ' ';
      put_int(s, remap[tris[3 * t + 2]] + 1);
      s += '\n';
    }
  });
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    ibf::set_error(std::string("ibf_export_obj: cannot open ") + path + ": " + std::strerror(errno));
    return IBF_ERR_IO;
  }
  // "\n".join(lines) + "\n" when there are lines: every line ends in "\n"
  bool ok = true;
  for (auto* parts : {&vparts, &fparts})
    for (auto& s : *parts)
      if (!s.empty()) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    ibf::set_error(std::string("ibf_export_obj: write failed on ") + path);
    return IBF_ERR_IO;
  }
  return IBF_OK;
}
