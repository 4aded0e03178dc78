// File formats either side of the hot path: the reference's
// ESRI ASCII grid (raster.cpp:22-96) and `.nug` text grid (quadgrid.cpp:287-
// 327), kept byte-compatible, plus a binary side format for both (a 67 M-value
// text DEM is ~1.3 GB and minutes of parsing; the binary one is one read into
// page-locked memory).  Host code only: nothing here touches the device
// except through the public grid calls (fm_grid_leaves / fm_grid_import).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "fm_internal.hpp"
#include "fm_io.hpp"

namespace fmh {
namespace {

constexpr char kRasterMagic[8] = {'F', 'M', 'R', 'B', '1', 0, 0, 0};
constexpr char kGridMagic[8] = {'F', 'M', 'N', 'G', '1', 0, 0, 0};

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
  File(const File&) = delete;
  File& operator=(const File&) = delete;
};

std::string slurp(const std::string& path, const char* what) {
  File in(path.c_str(), "rb");
  if (!in.f) throw Error(FM_ERR_IO, std::string("cannot open ") + what + " file: " + path);
  std::string s;
  if (std::fseek(in.f, 0, SEEK_END) == 0) {
    const long n = std::ftell(in.f);
    std::rewind(in.f);
    if (n > 0) s.resize(size_t(n));
    if (n > 0 && std::fread(&s[0], 1, size_t(n), in.f) != size_t(n))
      throw Error(FM_ERR_IO, "read failed: " + path);
  }
  return s;
}

inline bool is_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// One whitespace-separated number as `istream >> double` reads it: a decimal
// literal, optional sign and exponent, correctly rounded; "nan", "inf" and hex
// floats are not numbers to the reference's stream and end the sequence.
inline bool parse_double(const char*& p, const char* end, double& v) {
  while (p < end && is_space(*p)) ++p;
  if (p >= end) return false;
  const char* q = p;
  if (*q == '+') ++q;
  if (q >= end) return false;
  const char c = (*q == '-' && q + 1 < end) ? q[1] : *q;
  if (!((c >= '0' && c <= '9') || c == '.')) return false;
  const auto r = std::from_chars(q, end, v, std::chars_format::general);
  if (r.ec == std::errc::invalid_argument) return false;
  if (r.ec == std::errc::result_out_of_range) return false;  // the stream sets failbit too
  p = r.ptr;
  return true;
}

inline bool parse_int(const char*& p, const char* end, int& v) {
  while (p < end && is_space(*p)) ++p;
  if (p >= end) return false;
  const char* q = p;
  if (*q == '+') ++q;
  const auto r = std::from_chars(q, end, v, 10);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}

unsigned io_threads(size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return unsigned(std::max<size_t>(1, std::min<size_t>(hw, bytes >> 20)));
}

// `n` doubles in page-locked memory when a device is there (uploads at the
// host link's rate), plain memory otherwise.
double* alloc_values(size_t n) {
  void* p = std::malloc(std::max<size_t>(n, 1) * sizeof(double));
  if (!p) throw std::bad_alloc();
  if (cudaHostRegister(p, std::max<size_t>(n, 1) * sizeof(double), cudaHostRegisterDefault) != cudaSuccess)
    (void)cudaGetLastError();  // no device: the buffer stays pageable
  return static_cast<double*>(p);
}

std::string lower(std::string s) {
  for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

void write_all(const std::string& path, const char* what, const std::vector<std::string>& parts) {
  File out(path.c_str(), "wb");
  if (!out.f) throw Error(FM_ERR_IO, std::string("cannot write ") + what + " file: " + path);
  for (const std::string& s : parts)
    if (!s.empty() && std::fwrite(s.data(), 1, s.size(), out.f) != s.size())
      throw Error(FM_ERR_IO, "write failed: " + path);
  if (std::fflush(out.f) != 0) throw Error(FM_ERR_IO, "write failed: " + path);
}

// operator<< of a double at precision 17 with no floatfield flag = "%.17g",
// which to_chars(general, 17) is specified to reproduce
inline void put_g17(std::string& s, double v) {
  char buf[48];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 17);
  s.append(buf, size_t(r.ptr - buf));
}

template <typename T>
void put_raw(std::string& s, const T& v) {
  s.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get_raw(const std::string& s, size_t& off, const std::string& path) {
  if (off + sizeof(T) > s.size()) throw Error(FM_ERR_IO, path + ": truncated binary header");
  T v;
  std::memcpy(&v, s.data() + off, sizeof(T));
  off += sizeof(T);
  return v;
}

}  // namespace

void raster_release(fm_raster* r) {
  if (!r || !r->values) return;
  void* p = const_cast<double*>(r->values);
  if (cudaHostUnregister(p) != cudaSuccess) (void)cudaGetLastError();
  std::free(p);
  r->values = nullptr;
}

// read_ascii_grid (raster.cpp:22-79), or the binary side format by its magic.
void raster_read(const std::string& path, fm_raster* out) {
  const std::string buf = slurp(path, "raster");
  fm_raster r{};
  if (buf.size() >= 8 && std::memcmp(buf.data(), kRasterMagic, 8) == 0) {
    size_t off = 8;
    r.ncols = get_raw<int32_t>(buf, off, path);
    r.nrows = get_raw<int32_t>(buf, off, path);
    r.xll = get_raw<double>(buf, off, path);
    r.yll = get_raw<double>(buf, off, path);
    r.cellsize = get_raw<double>(buf, off, path);
    r.nodata = get_raw<double>(buf, off, path);
    if (r.ncols < 1 || r.nrows < 1 || !(r.cellsize > 0.0))
      throw Error(FM_ERR_IO, path + ": invalid raster dimensions in header");
    const size_t n = size_t(r.ncols) * size_t(r.nrows);
    const size_t have = (buf.size() - off) / sizeof(double);
    if ((buf.size() - off) != n * sizeof(double))
      throw Error(FM_ERR_IO, path + ": expected " + std::to_string(n) + " values, found " + std::to_string(have));
    double* v = alloc_values(n);
    std::memcpy(v, buf.data() + off, n * sizeof(double));
    r.values = v;
    *out = r;
    return;
  }

  // Header: six keyword/value lines in any order, keywords case-insensitive,
  // every value read as a double (raster.cpp:30-68).
  const char* p = buf.data();
  const char* const end = p + buf.size();
  bool have[6] = {false, false, false, false, false, false};
  for (int line_no = 1; line_no <= 6; ++line_no) {
    if (p >= end) throw Error(FM_ERR_IO, path + ": truncated header at line " + std::to_string(line_no));
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    const char* const line_end = eol ? eol : end;
    const std::string line(p, line_end);
    const char* q = p;
    while (q < line_end && is_space(*q)) ++q;
    const char* k0 = q;
    while (q < line_end && !is_space(*q)) ++q;
    std::string key(k0, q);
    double val = 0.0;
    if (key.empty() || !parse_double(q, line_end, val))
      throw Error(FM_ERR_IO,
                  path + ": malformed header line " + std::to_string(line_no) + ": \"" + line + "\"");
    key = lower(key);
    if (key == "ncols") {
      r.ncols = int(val);
      have[0] = true;
    } else if (key == "nrows") {
      r.nrows = int(val);
      have[1] = true;
    } else if (key == "xllcorner") {
      r.xll = val;
      have[2] = true;
    } else if (key == "yllcorner") {
      r.yll = val;
      have[3] = true;
    } else if (key == "cellsize") {
      r.cellsize = val;
      have[4] = true;
    } else if (key == "nodata_value") {
      r.nodata = val;
      have[5] = true;
    } else {
      throw Error(FM_ERR_IO, path + ": unknown header keyword at line " + std::to_string(line_no) + ": \"" +
                                 key + "\"");
    }
    p = eol ? eol + 1 : end;
  }
  for (int k = 0; k < 6; ++k)
    if (!have[k]) throw Error(FM_ERR_IO, path + ": incomplete six-keyword header");
  if (r.ncols < 1 || r.nrows < 1 || r.cellsize <= 0.0)
    throw Error(FM_ERR_IO, path + ": invalid raster dimensions in header");

  // Values: the body cut at whitespace into one slice per thread, each parsed
  // on its own; the sequence ends at the first token that is not a number
  // (`while (in >> v)`, raster.cpp:73), and its length must be ncols * nrows.
  const size_t n = size_t(r.ncols) * size_t(r.nrows);
  const unsigned T = io_threads(size_t(end - p));
  std::vector<const char*> cut(T + 1);
  cut[0] = p;
  cut[T] = end;
  for (unsigned t = 1; t < T; ++t) {
    const char* c = p + size_t(end - p) / T * t;
    c = std::max(c, cut[t - 1]);
    while (c < end && !is_space(*c)) ++c;
    cut[t] = c;
  }
  std::vector<std::vector<double>> part(T);
  std::vector<char> clean(T, 1);
  auto work = [&](unsigned t) {
    const char* a = cut[t];
    const char* const b = cut[t + 1];
    std::vector<double>& v = part[t];
    v.reserve(size_t(b - a) / 8 + 16);
    double x;
    while (parse_double(a, b, x)) v.push_back(x);
    while (a < b && is_space(*a)) ++a;
    clean[t] = (a >= b);
  };
  {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  size_t found = 0;
  unsigned used = 0;
  for (; used < T; ++used) {
    found += part[used].size();
    if (!clean[used]) {
      ++used;
      break;
    }
  }
  if (found != n)
    throw Error(FM_ERR_IO,
                path + ": expected " + std::to_string(n) + " values, found " + std::to_string(found));
  double* v = alloc_values(n);
  size_t off = 0;
  for (unsigned t = 0; t < used; ++t) {
    if (!part[t].empty()) std::memcpy(v + off, part[t].data(), part[t].size() * sizeof(double));
    off += part[t].size();
  }
  r.values = v;
  *out = r;
}

static void require_host_raster(const fm_raster* r) {
  if (!r || !r->values || r->ncols < 1 || r->nrows < 1) throw Error(FM_ERR_IO, "raster write: empty raster");
  if (r->on_device)
    throw Error(FM_ERR_IO, "raster write: the raster is device resident; download it first "
                           "(fm_sim_raster with out_on_device = 0)");
}

// write_ascii_grid (raster.cpp:81-96), byte for byte.
void raster_write_ascii(const fm_raster* r, const std::string& path) {
  require_host_raster(r);
  const size_t nr = size_t(r->nrows), nc = size_t(r->ncols);
  const unsigned T = unsigned(std::min<size_t>(io_threads(nr * nc * 8), nr));
  std::vector<std::string> parts(T + 1);
  std::string& h = parts[0];
  h += "ncols " + std::to_string(r->ncols) + "\nnrows " + std::to_string(r->nrows) + "\nxllcorner ";
  put_g17(h, r->xll);
  h += "\nyllcorner ";
  put_g17(h, r->yll);
  h += "\ncellsize ";
  put_g17(h, r->cellsize);
  h += "\nNODATA_value ";
  put_g17(h, r->nodata);
  h += "\n";
  auto work = [&](unsigned t) {
    const size_t r0 = nr * t / T, r1 = nr * (t + 1) / T;
    std::string& s = parts[t + 1];
    s.reserve((r1 - r0) * nc * 12);
    for (size_t row = r0; row < r1; ++row) {
      const double* v = r->values + row * nc;
      for (size_t col = 0; col < nc; ++col) {
        if (col) s.push_back(' ');
        put_g17(s, v[col]);
      }
      s.push_back('\n');
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  write_all(path, "raster", parts);
}

void raster_write_bin(const fm_raster* r, const std::string& path) {
  require_host_raster(r);
  std::vector<std::string> parts(2);
  std::string& h = parts[0];
  h.append(kRasterMagic, 8);
  put_raw(h, int32_t(r->ncols));
  put_raw(h, int32_t(r->nrows));
  put_raw(h, r->xll);
  put_raw(h, r->yll);
  put_raw(h, r->cellsize);
  put_raw(h, r->nodata);
  File out(path.c_str(), "wb");
  if (!out.f) throw Error(FM_ERR_IO, "cannot write raster file: " + path);
  const size_t n = size_t(r->ncols) * size_t(r->nrows);
  if (std::fwrite(h.data(), 1, h.size(), out.f) != h.size() ||
      std::fwrite(r->values, sizeof(double), n, out.f) != n || std::fflush(out.f) != 0)
    throw Error(FM_ERR_IO, "write failed: " + path);
}

// write_nug (quadgrid.cpp:287-302) in the reference's leaf order, byte for
// byte; binary != 0: the same fields raw.
void grid_write(const fm_grid* g, const std::string& path, bool binary) {
  int32_t L, M, N;
  double R, x0, y0, norm;
  if (fm_grid_info(g, &L, &M, &N, &R, &x0, &y0, &norm) != FM_OK) throw Error(FM_ERR_IO, fm_last_error());
  const int64_t n = fm_grid_num_leaves(g);
  const size_t nn = size_t(n);
  std::vector<int32_t> lv(nn), li(nn), lj(nn);
  std::vector<double> z(nn * 3);
  if (fm_grid_leaves(g, FM_ORDER_REFERENCE, lv.data(), li.data(), lj.data(), z.data()) != FM_OK)
    throw Error(FM_ERR_IO, fm_last_error());
  if (binary) {
    std::vector<std::string> parts(1);
    std::string& h = parts[0];
    h.append(kGridMagic, 8);
    put_raw(h, L);
    put_raw(h, M);
    put_raw(h, N);
    put_raw(h, int32_t(0));
    put_raw(h, R);
    put_raw(h, x0);
    put_raw(h, y0);
    put_raw(h, int64_t(n));
    h.append(reinterpret_cast<const char*>(lv.data()), size_t(n) * 4);
    h.append(reinterpret_cast<const char*>(li.data()), size_t(n) * 4);
    h.append(reinterpret_cast<const char*>(lj.data()), size_t(n) * 4);
    h.append(reinterpret_cast<const char*>(z.data()), size_t(n) * 24);
    write_all(path, "grid", parts);
    return;
  }
  const unsigned T = unsigned(std::max<int64_t>(1, std::min<int64_t>(io_threads(size_t(n) * 64), n)));
  std::vector<std::string> parts(T + 1);
  std::string& h = parts[0];
  h += "nug " + std::to_string(L) + " " + std::to_string(M) + " " + std::to_string(N) + " ";
  put_g17(h, R);
  h += " ";
  put_g17(h, x0);
  h += " ";
  put_g17(h, y0);
  h += "\n";
  auto work = [&](unsigned t) {
    const size_t k0 = size_t(n) * t / T, k1 = size_t(n) * (t + 1) / T;
    std::string& s = parts[t + 1];
    s.reserve((k1 - k0) * 72);
    for (size_t k = k0; k < k1; ++k) {
      s += std::to_string(lv[k]);
      s.push_back(' ');
      s += std::to_string(li[k]);
      s.push_back(' ');
      s += std::to_string(lj[k]);
      for (int q = 0; q < 3; ++q) {
        s.push_back(' ');
        put_g17(s, z[3 * k + q]);
      }
      s.push_back('\n');
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  write_all(path, "grid", parts);
}

// read_nug (quadgrid.cpp:304-327): header, then records until the first one
// that does not parse; make_quadgrid's checks are fm_grid_import's.
void grid_read(const std::string& path, fm_grid** out) {
  const std::string buf = slurp(path, "grid");
  int32_t L, M, N;
  double R, x0, y0;
  std::vector<int32_t> lv, li, lj;
  std::vector<double> z;
  if (buf.size() >= 8 && std::memcmp(buf.data(), kGridMagic, 8) == 0) {
    size_t off = 8;
    L = get_raw<int32_t>(buf, off, path);
    M = get_raw<int32_t>(buf, off, path);
    N = get_raw<int32_t>(buf, off, path);
    (void)get_raw<int32_t>(buf, off, path);
    R = get_raw<double>(buf, off, path);
    x0 = get_raw<double>(buf, off, path);
    y0 = get_raw<double>(buf, off, path);
    const int64_t n = get_raw<int64_t>(buf, off, path);
    if (n < 0 || (buf.size() - off) / 36 < size_t(n) || buf.size() - off != size_t(n) * 36)
      throw Error(FM_ERR_IO, path + ": malformed binary grid (leaf count does not match the file size)");
    lv.resize(size_t(n));
    li.resize(size_t(n));
    lj.resize(size_t(n));
    z.resize(size_t(n) * 3);
    std::memcpy(lv.data(), buf.data() + off, size_t(n) * 4);
    std::memcpy(li.data(), buf.data() + off + size_t(n) * 4, size_t(n) * 4);
    std::memcpy(lj.data(), buf.data() + off + size_t(n) * 8, size_t(n) * 4);
    std::memcpy(z.data(), buf.data() + off + size_t(n) * 12, size_t(n) * 24);
  } else {
    const char* p = buf.data();
    const char* const end = p + buf.size();
    while (p < end && is_space(*p)) ++p;
    const char* m0 = p;
    while (p < end && !is_space(*p)) ++p;
    const std::string magic(m0, p);
    if (magic != "nug" || !parse_int(p, end, L) || !parse_int(p, end, M) || !parse_int(p, end, N) ||
        !parse_double(p, end, R) || !parse_double(p, end, x0) || !parse_double(p, end, y0))
      throw Error(FM_ERR_IO, path + ": malformed .nug header");
    for (;;) {
      int a, b, c;
      double d[3];
      if (!parse_int(p, end, a) || !parse_int(p, end, b) || !parse_int(p, end, c) ||
          !parse_double(p, end, d[0]) || !parse_double(p, end, d[1]) || !parse_double(p, end, d[2]))
        break;
      lv.push_back(a);
      li.push_back(b);
      lj.push_back(c);
      z.insert(z.end(), d, d + 3);
    }
  }
  const int st = fm_grid_import(L, M, N, R, x0, y0, int64_t(lv.size()), lv.data(), li.data(), lj.data(),
                                z.data(), out);
  if (st != FM_OK) throw Error(st, path + ": " + fm_last_error());
}

}  // namespace fmh
