// Native writers of the mesh output formats:
// legacy-VTK structured grids (write_mesh_vtk, ddmesh/fileio.py:45-68) and
// report CSVs are ASCII with 17 significant digits.  At BASELINE sizes
// (C3: 16.8 M nodes, C5: 135 M) the reference's per-row Python formatting
// dominates a solve's output time; here the rows are formatted by a pool of
// host threads into per-chunk buffers and written in order.  The bytes are
// identical to the reference writer's (printf "%.17g" is correctly rounded,
// as is Python's formatting; NaN/inf are spelled as Python spells them).

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ddpma.h"

namespace {

// Python's f"{v:.17g}" for one double, appended to out.
inline void fmt17(std::string& out, double v) {
  char buf[40];
  int n;
  if (std::isnan(v)) {
    n = snprintf(buf, sizeof buf, "nan");
  } else if (std::isinf(v)) {
    n = snprintf(buf, sizeof buf, v > 0 ? "inf" : "-inf");
  } else {
    n = snprintf(buf, sizeof buf, "%.17g", v);
  }
  out.append(buf, (size_t)n);
}

// Format rows [0, n) with fn(i, out) on up to `threads` threads, in order.
template <class F>
bool write_rows(FILE* fp, long long n, const F& fn) {
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const long long chunk = 1 << 16;
  const long long nchunks = (n + chunk - 1) / chunk;
  const int T = (int)std::min<long long>(hw, std::max<long long>(1, nchunks));
  // process in waves of T chunks so memory stays bounded
  std::vector<std::string> bufs(T);
  for (long long c0 = 0; c0 < nchunks; c0 += T) {
    const int nw = (int)std::min<long long>(T, nchunks - c0);
    std::vector<std::thread> pool;
    for (int t = 0; t < nw; ++t) {
      pool.emplace_back([&, t] {
        std::string& s = bufs[t];
        s.clear();
        const long long b = (c0 + t) * chunk, e = std::min(n, b + chunk);
        s.reserve((size_t)(e - b) * 64);
        for (long long i = b; i < e; ++i) fn(i, s);
      });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < nw; ++t)
      if (fwrite(bufs[t].data(), 1, bufs[t].size(), fp) != bufs[t].size()) return false;
  }
  return true;
}

thread_local std::string g_io_err;

}  // namespace

extern "C" const char* ddpma_io_error(void) { return g_io_err.c_str(); }

extern "C" ddpma_status ddpma_write_mesh_vtk(const char* path, int dim, const int* counts,
                                             const double* coords, const double* jac,
                                             const double* e_adp, const char* title,
                                             const char* first_scalar) {
  if (dim != 2 && dim != 3) {
    g_io_err = "dim must be 2 or 3";
    return DDPMA_ERR_CONFIG;
  }
  FILE* fp = fopen(path, "wb");
  if (!fp) {
    g_io_err = std::string("cannot open ") + path;
    return DDPMA_ERR_IO;
  }
  const long long n0 = counts[0], n1 = counts[1], n2 = dim == 3 ? counts[2] : 1;
  const long long n = n0 * n1 * n2;
  std::string head;
  head += "# vtk DataFile Version 3.0\n";
  head += title;
  head += "\nASCII\nDATASET STRUCTURED_GRID\n";
  head += "DIMENSIONS " + std::to_string(n0) + " " + std::to_string(n1) + " " +
          std::to_string(n2) + "\n";
  head += "POINTS " + std::to_string(n) + " double\n";
  bool ok = fwrite(head.data(), 1, head.size(), fp) == head.size();
  // x varies fastest (ravel(order="F")): flat index i -> (i0, i1, i2) with
  // i0 fastest; the C-order source index is (i0*n1 + i1)*n2 + i2.
  auto src = [&](long long i) {
    const long long i0 = i % n0, r = i / n0, i1 = r % n1, i2 = r / n1;
    return (i0 * n1 + i1) * n2 + i2;
  };
  if (ok)
    ok = write_rows(fp, n, [&](long long i, std::string& s) {
      const long long k = src(i);
      for (int q = 0; q < 3; ++q) {
        fmt17(s, q < dim ? coords[k * dim + q] : 0.0);
        s.push_back(q < 2 ? ' ' : '\n');
      }
    });
  const double* fields[2] = {jac, e_adp};
  const char* names[2] = {first_scalar, "e_adp"};
  if (ok) {
    const std::string pd = "POINT_DATA " + std::to_string(n) + "\n";
    ok = fwrite(pd.data(), 1, pd.size(), fp) == pd.size();
  }
  for (int f = 0; f < 2 && ok; ++f) {
    if (!fields[f]) continue;
    const std::string h = std::string("SCALARS ") + names[f] + " double\nLOOKUP_TABLE default\n";
    ok = fwrite(h.data(), 1, h.size(), fp) == h.size();
    const double* v = fields[f];
    if (ok)
      ok = write_rows(fp, n, [&](long long i, std::string& s) {
        fmt17(s, v[src(i)]);
        s.push_back('\n');
      });
  }
  if (fclose(fp) != 0) ok = false;
  if (!ok) {
    g_io_err = std::string("write failed: ") + path;
    return DDPMA_ERR_IO;
  }
  return DDPMA_OK;
}
