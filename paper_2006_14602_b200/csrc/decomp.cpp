// Overlapping slab/block decomposition — host-side restatement of
// ddmesh/grid.py:125-258 (build_decomposition, _partition_axis, _extend_axis,
// _check_decomposition).  Index ranges, ids, faces and donors are bit-exact
// with the reference; error messages are the reference's strings.
//
// Pure host code (no CUDA): callable from the CPU test-suite.

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ddpma.h"
#include "ddpma_internal.h"

namespace ddpma {

static thread_local std::string g_err;

void set_global_error(const std::string& s) { g_err = s; }
const char* global_error() { return g_err.c_str(); }

namespace {

struct Seg { int lo, hi; };

// grid.py:125-135 — near-equal disjoint partition, remainder to low parts.
std::vector<Seg> partition_axis(int n, int parts) {
  std::vector<Seg> out;
  int base = n / parts, rem = n % parts, start = 0;
  for (int p = 0; p < parts; ++p) {
    int size = base + (p < rem ? 1 : 0);
    out.push_back({start, start + size - 1});
    start += size;
  }
  return out;
}

// grid.py:138-173 — extend into neighbours; midline ownership cuts.
bool extend_axis(const std::vector<Seg>& segs, int overlap, int n, int axis,
                 std::vector<Seg>& boxes, std::vector<int>& cuts) {
  const int up = overlap / 2;      // Python floor division; overlap >= 2 here
  const int down = overlap - up;
  const int m = (int)segs.size();
  boxes.clear();
  cuts.clear();
  for (int p = 0; p < m; ++p) {
    int lo = p > 0 ? segs[p].lo - down : segs[p].lo;
    int hi = p < m - 1 ? segs[p].hi + up : segs[p].hi;
    boxes.push_back({lo, hi});
  }
  for (int p = 0; p + 1 < m; ++p) {
    int a = boxes[p + 1].lo, b = boxes[p].hi;
    int s = a + b;
    cuts.push_back(s >= 0 ? s / 2 : -((-s + 1) / 2));  // Python //, floor
  }
  char buf[256];
  for (int p = 0; p + 1 < m; ++p) {
    int lo0 = boxes[p].lo, hi0 = boxes[p].hi, lo1 = boxes[p + 1].lo, hi1 = boxes[p + 1].hi;
    if (!(lo0 < lo1 && lo1 < hi0 && hi0 < hi1)) {
      snprintf(buf, sizeof buf,
               "overlap %d too large for %d nodes split %d ways along axis %d",
               overlap, n, m, axis);
      set_global_error(buf);
      return false;
    }
  }
  for (int p = 0; p + 2 < m; ++p) {
    if (boxes[p + 2].lo <= boxes[p].hi) {
      snprintf(buf, sizeof buf,
               "overlap %d makes non-adjacent boxes touch along axis %d", overlap, axis);
      set_global_error(buf);
      return false;
    }
  }
  for (auto& b : boxes) {
    if (b.hi - b.lo + 1 < 3) {
      snprintf(buf, sizeof buf, "axis %d: a subdomain box has fewer than 3 nodes", axis);
      set_global_error(buf);
      return false;
    }
  }
  return true;
}

std::string tuple_str(const int* v, int n) {
  std::string s = "(";
  for (int i = 0; i < n; ++i) {
    s += std::to_string(v[i]);
    if (n == 1) s += ",";
    else if (i + 1 < n) s += ", ";
  }
  return s + ")";
}

}  // namespace

}  // namespace ddpma

using namespace ddpma;

extern "C" const char* ddpma_global_error(void) { return global_error(); }

extern "C" ddpma_status ddpma_build_decomposition(int dim, const int* counts,
                                                  const int* layout, int overlap,
                                                  ddpma_subdomain* out, int cap,
                                                  int* nsub) {
  char buf[256];
  if (dim < 1 || dim > 3) {
    set_global_error("dim must be 2 or 3");
    return DDPMA_ERR_CONFIG;
  }
  // grid.py:185-191
  for (int k = 0; k < dim; ++k) {
    if (layout[k] < 1) {
      set_global_error("layout parts must be >= 1, got " + tuple_str(layout, dim));
      return DDPMA_ERR_CONFIG;
    }
  }
  bool split = false;
  for (int k = 0; k < dim; ++k) split |= layout[k] > 1;
  if (split && overlap < 2) {
    snprintf(buf, sizeof buf, "overlap must be >= 2, got %d", overlap);
    set_global_error(buf);
    return DDPMA_ERR_CONFIG;
  }
  std::vector<Seg> axis_boxes[3], axis_owned[3];
  for (int k = 0; k < dim; ++k) {
    const int n = counts[k];
    std::vector<int> cuts;
    if (layout[k] == 1) {
      axis_boxes[k] = {{0, n - 1}};
    } else if (!extend_axis(partition_axis(n, layout[k]), overlap, n, k, axis_boxes[k], cuts)) {
      return DDPMA_ERR_CONFIG;
    }
    // grid.py:206-209: bounds = [-1] + cuts + [n-1]
    std::vector<int> bounds{-1};
    bounds.insert(bounds.end(), cuts.begin(), cuts.end());
    bounds.push_back(n - 1);
    for (int p = 0; p < layout[k]; ++p) axis_owned[k].push_back({bounds[p] + 1, bounds[p + 1]});
  }
  // _check_decomposition (grid.py:240-258) factorises over axes for a tensor
  // product of boxes: coverage and the ownership partition hold globally iff
  // they hold per axis, which is what is checked here (no global int arrays).
  for (int k = 0; k < dim; ++k) {
    int covered_to = -1;
    for (auto& b : axis_boxes[k]) {
      if (b.lo > covered_to + 1) {
        set_global_error("decomposition does not cover the grid");
        return DDPMA_ERR_CONFIG;
      }
      if (b.hi > covered_to) covered_to = b.hi;
    }
    if (covered_to < counts[k] - 1) {
      set_global_error("decomposition does not cover the grid");
      return DDPMA_ERR_CONFIG;
    }
    int expect = 0;
    for (auto& o : axis_owned[k]) {
      if (o.lo != expect || o.hi < o.lo) {
        set_global_error("node ownership is not a partition");
        return DDPMA_ERR_CONFIG;
      }
      expect = o.hi + 1;
    }
    if (expect != counts[k]) {
      set_global_error("node ownership is not a partition");
      return DDPMA_ERR_CONFIG;
    }
  }
  int total = 1;
  for (int k = 0; k < dim; ++k) total *= layout[k];
  *nsub = total;
  std::vector<ddpma_subdomain> subs(total);
  // itertools.product order: last axis fastest (grid.py:211-212)
  for (int i = 0; i < total; ++i) {
    ddpma_subdomain& s = subs[i];
    memset(&s, 0, sizeof s);
    s.id = i;
    int rem = i;
    for (int k = dim - 1; k >= 0; --k) {
      s.pos[k] = rem % layout[k];
      rem /= layout[k];
    }
    for (int k = 0; k < dim; ++k) {
      s.box[k][0] = axis_boxes[k][s.pos[k]].lo;
      s.box[k][1] = axis_boxes[k][s.pos[k]].hi;
      s.owned[k][0] = axis_owned[k][s.pos[k]].lo;
      s.owned[k][1] = axis_owned[k][s.pos[k]].hi;
      s.face[k][0] = s.pos[k] == 0 ? DDPMA_FACE_PHYSICAL : DDPMA_FACE_INTERFACE;
      s.face[k][1] = s.pos[k] == layout[k] - 1 ? DDPMA_FACE_PHYSICAL : DDPMA_FACE_INTERFACE;
      int stride = 1;
      for (int q = dim - 1; q > k; --q) stride *= layout[q];
      s.donor[k][0] = s.face[k][0] == DDPMA_FACE_INTERFACE ? i - stride : -1;
      s.donor[k][1] = s.face[k][1] == DDPMA_FACE_INTERFACE ? i + stride : -1;
    }
    for (int k = dim; k < 3; ++k) {
      s.donor[k][0] = s.donor[k][1] = -1;
    }
  }
  // trace lines strictly interior to the donor (grid.py:251-258)
  for (auto& s : subs) {
    for (int k = 0; k < dim; ++k) {
      for (int side = 0; side < 2; ++side) {
        int d = s.donor[k][side];
        if (d < 0) continue;
        int line = s.box[k][side];
        int nlo = subs[d].box[k][0], nhi = subs[d].box[k][1];
        if (!(nlo < line && line < nhi)) {
          snprintf(buf, sizeof buf,
                   "trace line %d of subdomain %d is not interior to donor %d (axis %d)",
                   line, s.id, d, k);
          set_global_error(buf);
          return DDPMA_ERR_CONFIG;
        }
      }
    }
  }
  if (out != nullptr && cap >= total) memcpy(out, subs.data(), sizeof(ddpma_subdomain) * total);
  return DDPMA_OK;
}

// integrate.py:77-106 — damped RKC2 coefficients (host scalar arithmetic in
// the reference's evaluation order; compiled with -ffp-contract=off).
extern "C" int ddpma_alternating_levels(int dim, const ddpma_subdomain* subs, int nsub, int* level) {
  int nlev = 0;
  for (int i = 0; i < nsub; ++i) {
    int lev = 0;
    for (int m = 0; m < i; ++m) {
      bool nb = false;
      for (int k = 0; k < dim; ++k)
        for (int side = 0; side < 2; ++side)
          nb = nb || subs[i].donor[k][side] == m || subs[m].donor[k][side] == i;
      if (nb && level[m] + 1 > lev) lev = level[m] + 1;
    }
    level[i] = lev;
    if (lev + 1 > nlev) nlev = lev + 1;
  }
  return nlev;
}

extern "C" ddpma_status ddpma_rkc_coeffs(int s, double* w0o, double* w1o, double* mu1to,
                                         double* mu, double* nu, double* mut, double* gt) {
  if (s < 2) {
    set_global_error("RKC2 needs at least 2 stages");
    return DDPMA_ERR_CONFIG;
  }
  RkcCoeffs c;
  rkc_coeffs(s, c);
  *w0o = c.w0;
  *w1o = c.w1;
  *mu1to = c.mu1t;
  for (int j = 0; j <= s; ++j) {
    mu[j] = c.mu[j];
    nu[j] = c.nu[j];
    mut[j] = c.mut[j];
    gt[j] = c.gt[j];
  }
  return DDPMA_OK;
}

namespace ddpma {

void rkc_coeffs(int s, RkcCoeffs& out) {
  const double damping = 2.0 / 13.0;
  const double w0 = 1.0 + damping / (double)(s * s);
  std::vector<double> t(s + 1), dt(s + 1), d2t(s + 1);
  t[0] = 1.0;
  t[1] = w0;
  dt[0] = 0.0;
  dt[1] = 1.0;
  d2t[0] = 0.0;
  d2t[1] = 0.0;
  for (int j = 2; j <= s; ++j) {
    t[j] = 2.0 * w0 * t[j - 1] - t[j - 2];
    dt[j] = 2.0 * w0 * dt[j - 1] - dt[j - 2] + 2.0 * t[j - 1];
    d2t[j] = 2.0 * w0 * d2t[j - 1] - d2t[j - 2] + 4.0 * dt[j - 1];
  }
  const double w1 = dt[s] / d2t[s];
  std::vector<double> b(s + 1), a(s + 1);
  for (int j = 2; j <= s; ++j) b[j] = d2t[j] / (dt[j] * dt[j]);
  b[0] = b[1] = b[2];
  for (int j = 0; j <= s; ++j) a[j] = 1.0 - b[j] * t[j];
  out.w0 = w0;
  out.w1 = w1;
  out.mu1t = b[1] * w1;
  out.mu.assign(s + 1, 0.0);
  out.nu.assign(s + 1, 0.0);
  out.mut.assign(s + 1, 0.0);
  out.gt.assign(s + 1, 0.0);
  for (int j = 2; j <= s; ++j) {
    out.mu[j] = 2.0 * b[j] * w0 / b[j - 1];
    out.nu[j] = -b[j] / b[j - 2];
    out.mut[j] = out.mu[j] * w1 / w0;
    out.gt[j] = -a[j - 1] * out.mut[j];
  }
}

}  // namespace ddpma
