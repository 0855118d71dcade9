// Slicing planner: tile-grid index arithmetic + per-rank op generation.
//
// Integer-only C++ restatement of
//   tiling.py:125-221  (most_square_grid, grid_shape, tile_bounds,
//                       overlapping_tiles, intersect, owner_of)
//   distmatrix.py:75-122 (replica placement, owned_tiles)
//   opgen.py:57-200    (restrict_for_replication, global_to_local, _make_op,
//                       generate_stationary_{a,b,c}, generate)
//   runtime.py:89-93   (iteration_offset)
// The emitted op rows are identical, in content and order, to the
// reference's opgen.generate (checked against golden dumps in tests/).
// math.ceil(a / b) in the reference is exact below 2**53; here it is the
// integer ceil-div.
#include <cstdint>
#include <string>
#include <vector>

#include "um_internal.h"

namespace um {
namespace plan {

struct Range {
  int64_t lo, hi;
  int64_t len() const { return hi - lo; }
};

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// tiling.intersect (tiling.py:193-199): canonical empty range [lo,lo).
static inline Range intersect(Range a, Range b) {
  const int64_t lo = a.lo > b.lo ? a.lo : b.lo;
  const int64_t hi = a.hi < b.hi ? a.hi : b.hi;
  if (lo >= hi) return {lo, lo};
  return {lo, hi};
}

struct Mat {
  um_mat_desc d;
  int64_t gr, gc;   // tile grid (tiling.grid_shape, tiling.py:158-163)
  int64_t rpr;      // ranks per replica (distmatrix.py:83)
  int64_t tppr, tppc;

  Range tile_rows(int64_t i) const {  // tiling.tile_bounds rows (tiling.py:166-175)
    const int64_t lo = i * d.tile_rows;
    const int64_t hi = (i + 1) * d.tile_rows < d.rows ? (i + 1) * d.tile_rows : d.rows;
    return {lo, hi};
  }
  Range tile_cols(int64_t j) const {
    const int64_t lo = j * d.tile_cols;
    const int64_t hi = (j + 1) * d.tile_cols < d.cols ? (j + 1) * d.tile_cols : d.cols;
    return {lo, hi};
  }
  // tiling.owner_of + replica offset (tiling.py:206-221, distmatrix.py:109-114)
  int64_t owner_rank(int64_t i, int64_t j, int64_t replica) const {
    int64_t local;
    if (d.mapping == UM_BLOCK_CYCLIC)
      local = (i % d.grid_pr) * d.grid_pc + (j % d.grid_pc);
    else
      local = (i / tppr) * d.grid_pc + (j / tppc);
    return local + replica * rpr;
  }
  int64_t replica_of(int64_t rank) const { return rank / rpr; }  // distmatrix.py:106-107
  // tiling.overlapping_tiles index ranges (tiling.py:178-190); caller checks area > 0.
  void overlap(Range rows, Range cols, int64_t& i_lo, int64_t& i_hi, int64_t& j_lo, int64_t& j_hi) const {
    i_lo = rows.lo / d.tile_rows;
    i_hi = ceil_div(rows.hi, d.tile_rows);
    if (i_hi > gr) i_hi = gr;
    j_lo = cols.lo / d.tile_cols;
    j_hi = ceil_div(cols.hi, d.tile_cols);
    if (j_hi > gc) j_hi = gc;
  }
};

static int make_mat(const um_mat_desc* in, int64_t p, const char* name, Mat& out) {
  if (!in) return fail(UM_EVALUE, std::string("null descriptor ") + name);
  const um_mat_desc& d = *in;
  if (d.rows < 0 || d.cols < 0) return fail(UM_EVALUE, std::string("negative shape for ") + name);
  if (d.tile_rows < 1 || d.tile_cols < 1)
    return fail(UM_ECONFIG, std::string("tile shape must be >= 1x1 for ") + name);       // tiling.py:116-117
  if (d.grid_pr < 1 || d.grid_pc < 1)
    return fail(UM_ECONFIG, std::string("process grid must be >= 1x1 for ") + name);     // tiling.py:118-119
  if (d.c < 1 || p % d.c != 0)
    return fail(UM_ECONFIG, std::string("replication factor must divide process count for ") + name);  // distmatrix.py:75-76
  if (d.grid_pr * d.grid_pc != p / d.c)
    return fail(UM_ECONFIG, std::string("process grid does not cover the ranks of one replica for ") + name);  // distmatrix.py:78-82
  if (d.mapping != UM_BLOCK && d.mapping != UM_BLOCK_CYCLIC) return fail(UM_EVALUE, "bad mapping");
  out.d = d;
  out.gr = ceil_div(d.rows, d.tile_rows);
  out.gc = ceil_div(d.cols, d.tile_cols);
  out.rpr = p / d.c;
  out.tppr = ceil_div(out.gr, d.grid_pr);
  out.tppc = ceil_div(out.gc, d.grid_pc);
  if (out.tppr < 1) out.tppr = 1;  // empty grid: never used for division by a real tile
  if (out.tppc < 1) out.tppc = 1;
  return UM_OK;
}

// opgen.restrict_for_replication (opgen.py:57-68)
static Range restrict_for_replication(Range inner, int64_t c, int64_t r) {
  const int64_t step = inner.len() / c;
  const int64_t lo = inner.lo + r * step;
  const int64_t hi = (r == c - 1) ? inner.hi : lo + step;
  return {lo, hi};
}

struct Emitter {
  std::vector<int64_t> rows;
  bool ok = true;
  std::string err;

  // opgen._make_op + global_to_local (opgen.py:71-103)
  void emit(const Mat& A, const Mat& B, const Mat& C, int64_t ai, int64_t aj, int64_t bi, int64_t bj, int64_t ci,
            int64_t cj, Range m, Range k, Range n) {
    const Range ar = A.tile_rows(ai), ac = A.tile_cols(aj);
    const Range br = B.tile_rows(bi), bc = B.tile_cols(bj);
    const Range cr = C.tile_rows(ci), cc = C.tile_cols(cj);
    auto contains = [](Range t, Range g) { return t.lo <= g.lo && g.hi <= t.hi; };
    if (!contains(ar, m) || !contains(ac, k) || !contains(br, k) || !contains(bc, n) || !contains(cr, m) ||
        !contains(cc, n)) {
      ok = false;
      err = "op bounds not contained in tile";
      return;
    }
    const int64_t row[UM_OP_FIELDS] = {ai, aj, bi, bj, ci, cj, m.lo, m.hi, k.lo, k.hi, n.lo, n.hi,
                                       m.lo - ar.lo, m.hi - ar.lo, k.lo - ac.lo, k.hi - ac.lo,
                                       k.lo - br.lo, k.hi - br.lo, n.lo - bc.lo, n.hi - bc.lo,
                                       m.lo - cr.lo, m.hi - cr.lo, n.lo - cc.lo, n.hi - cc.lo};
    rows.insert(rows.end(), row, row + UM_OP_FIELDS);
  }
};

// opgen.generate_stationary_c (opgen.py:106-131)
static void gen_c(const Mat& A, const Mat& B, const Mat& C, int64_t caller, Emitter& e) {
  const int64_t k = A.d.cols;
  const Range ks = restrict_for_replication({0, k}, C.d.c, C.replica_of(caller));
  const int64_t rep = C.replica_of(caller);
  for (int64_t ci = 0; ci < C.gr; ++ci)
    for (int64_t cj = 0; cj < C.gc; ++cj) {
      if (C.owner_rank(ci, cj, rep) != caller) continue;
      const Range cr = C.tile_rows(ci), cc = C.tile_cols(cj);
      if (cr.len() * ks.len() == 0) continue;
      int64_t ai0, ai1, aj0, aj1;
      A.overlap(cr, ks, ai0, ai1, aj0, aj1);
      for (int64_t ai = ai0; ai < ai1; ++ai)
        for (int64_t aj = aj0; aj < aj1; ++aj) {
          const Range ar = A.tile_rows(ai), ac = A.tile_cols(aj);
          const Range k_in_a = intersect(ac, ks);
          if (k_in_a.len() * cc.len() == 0) continue;
          int64_t bi0, bi1, bj0, bj1;
          B.overlap(k_in_a, cc, bi0, bi1, bj0, bj1);
          for (int64_t bi = bi0; bi < bi1; ++bi)
            for (int64_t bj = bj0; bj < bj1; ++bj) {
              const Range br = B.tile_rows(bi), bc = B.tile_cols(bj);
              const Range m = intersect(cr, ar), kk = intersect(k_in_a, br), n = intersect(bc, cc);
              if (m.len() == 0 || kk.len() == 0 || n.len() == 0) continue;
              e.emit(A, B, C, ai, aj, bi, bj, ci, cj, m, kk, n);
            }
        }
    }
}

// opgen.generate_stationary_b (opgen.py:134-159)
static void gen_b(const Mat& A, const Mat& B, const Mat& C, int64_t caller, Emitter& e) {
  const int64_t m = A.d.rows;
  const Range ms = restrict_for_replication({0, m}, B.d.c, B.replica_of(caller));
  const int64_t rep = B.replica_of(caller);
  for (int64_t bi = 0; bi < B.gr; ++bi)
    for (int64_t bj = 0; bj < B.gc; ++bj) {
      if (B.owner_rank(bi, bj, rep) != caller) continue;
      const Range br = B.tile_rows(bi), bc = B.tile_cols(bj);
      if (ms.len() * br.len() == 0) continue;
      int64_t ai0, ai1, aj0, aj1;
      A.overlap(ms, br, ai0, ai1, aj0, aj1);
      for (int64_t ai = ai0; ai < ai1; ++ai)
        for (int64_t aj = aj0; aj < aj1; ++aj) {
          const Range ar = A.tile_rows(ai), ac = A.tile_cols(aj);
          const Range m_in_a = intersect(ar, ms);
          if (m_in_a.len() * bc.len() == 0) continue;
          int64_t ci0, ci1, cj0, cj1;
          C.overlap(m_in_a, bc, ci0, ci1, cj0, cj1);
          for (int64_t ci = ci0; ci < ci1; ++ci)
            for (int64_t cj = cj0; cj < cj1; ++cj) {
              const Range cr = C.tile_rows(ci), cc = C.tile_cols(cj);
              const Range mm = intersect(m_in_a, cr), k = intersect(ac, br), n = intersect(bc, cc);
              if (mm.len() == 0 || k.len() == 0 || n.len() == 0) continue;
              e.emit(A, B, C, ai, aj, bi, bj, ci, cj, mm, k, n);
            }
        }
    }
}

// opgen.generate_stationary_a (opgen.py:162-183)
static void gen_a(const Mat& A, const Mat& B, const Mat& C, int64_t caller, Emitter& e) {
  const int64_t n = B.d.cols;
  const Range ns = restrict_for_replication({0, n}, A.d.c, A.replica_of(caller));
  const int64_t rep = A.replica_of(caller);
  for (int64_t ai = 0; ai < A.gr; ++ai)
    for (int64_t aj = 0; aj < A.gc; ++aj) {
      if (A.owner_rank(ai, aj, rep) != caller) continue;
      const Range ar = A.tile_rows(ai), ac = A.tile_cols(aj);
      if (ac.len() * ns.len() == 0) continue;
      int64_t bi0, bi1, bj0, bj1;
      B.overlap(ac, ns, bi0, bi1, bj0, bj1);
      for (int64_t bi = bi0; bi < bi1; ++bi)
        for (int64_t bj = bj0; bj < bj1; ++bj) {
          const Range br = B.tile_rows(bi), bc = B.tile_cols(bj);
          const Range n_in_b = intersect(bc, ns);
          if (ar.len() * n_in_b.len() == 0) continue;
          int64_t ci0, ci1, cj0, cj1;
          C.overlap(ar, n_in_b, ci0, ci1, cj0, cj1);
          for (int64_t ci = ci0; ci < ci1; ++ci)
            for (int64_t cj = cj0; cj < cj1; ++cj) {
              const Range cr = C.tile_rows(ci), cc = C.tile_cols(cj);
              const Range m = intersect(cr, ar), k = intersect(ac, br), nn = intersect(n_in_b, cc);
              if (m.len() == 0 || k.len() == 0 || nn.len() == 0) continue;
              e.emit(A, B, C, ai, aj, bi, bj, ci, cj, m, k, nn);
            }
        }
    }
}

}  // namespace plan
}  // namespace um

using namespace um;
using namespace um::plan;

extern "C" int um_plan(const um_mat_desc* Ad, const um_mat_desc* Bd, const um_mat_desc* Cd, int32_t nprocs,
                       int32_t stationarity, int32_t caller, int64_t* ops_out, int64_t cap, int64_t* n_out) {
  if (nprocs < 1) return fail(UM_EVALUE, "need at least one process");
  Mat A, B, C;
  int rc;
  if ((rc = make_mat(Ad, nprocs, "A", A)) || (rc = make_mat(Bd, nprocs, "B", B)) || (rc = make_mat(Cd, nprocs, "C", C)))
    return rc;
  // opgen._check_shapes (opgen.py:81-89)
  if (A.d.cols != B.d.rows || A.d.rows != C.d.rows || B.d.cols != C.d.cols)
    return fail(UM_ECONFIG, "shapes do not conform: A " + std::to_string(A.d.rows) + "x" + std::to_string(A.d.cols) +
                                ", B " + std::to_string(B.d.rows) + "x" + std::to_string(B.d.cols) + ", C " +
                                std::to_string(C.d.rows) + "x" + std::to_string(C.d.cols));
  if (caller < 0 || caller >= nprocs) return fail(UM_EINDEX, "caller rank out of range");
  Emitter e;
  switch (stationarity) {
    case UM_STATIONARY_A: gen_a(A, B, C, caller, e); break;
    case UM_STATIONARY_B: gen_b(A, B, C, caller, e); break;
    case UM_STATIONARY_C: gen_c(A, B, C, caller, e); break;
    default: return fail(UM_EVALUE, "unknown stationarity");
  }
  if (!e.ok) return fail(UM_ECONTRACT, e.err);
  const int64_t n = (int64_t)(e.rows.size() / UM_OP_FIELDS);
  if (n_out) *n_out = n;
  if (n > cap) return fail(UM_ECAPACITY, "op buffer too small");
  if (n > 0) {
    if (!ops_out) return fail(UM_EVALUE, "null op buffer");
    for (size_t i = 0; i < e.rows.size(); ++i) ops_out[i] = e.rows[i];
  }
  return UM_OK;
}

extern "C" int um_iteration_offset(int64_t ti, int64_t tj, int64_t nops, int64_t* out) {
  if (nops < 1) return fail(UM_EVALUE, "nops must be >= 1");  // runtime.py:91-92
  if (!out) return fail(UM_EVALUE, "null out pointer");
  *out = (ti + tj) % nops;
  return UM_OK;
}

extern "C" int um_owner_rank(const um_mat_desc* M, int32_t nprocs, int64_t i, int64_t j, int32_t replica,
                             int32_t* rank_out) {
  Mat m;
  int rc;
  if ((rc = make_mat(M, nprocs, "M", m))) return rc;
  if (replica < 0 || replica >= M->c) return fail(UM_EINDEX, "replica out of range");      // distmatrix.py:111-112
  if (i < 0 || i >= m.gr || j < 0 || j >= m.gc) return fail(UM_EINDEX, "tile outside grid");  // tiling.py:216-217
  if (!rank_out) return fail(UM_EVALUE, "null out pointer");
  *rank_out = (int32_t)m.owner_rank(i, j, replica);
  return UM_OK;
}

extern "C" int um_most_square_grid(int64_t p, int64_t* gr, int64_t* gc) {
  if (p < 1) return fail(UM_EVALUE, "p must be >= 1");
  int64_t best = 1;
  for (int64_t d = 1; d * d <= p; ++d)
    if (p % d == 0) best = d;  // tiling.py:132-135: largest divisor <= isqrt(p)
  if (gr) *gr = best;
  if (gc) *gc = p / best;
  return UM_OK;
}
