// Host model: see od_model.hpp.  Compiled with -ffp-contract=off so that no
// multiply-add is fused differently from the reference build.
#include "od_model.hpp"

#include <algorithm>
#include <array>
#include <cmath>

namespace odb {

// ---------------------------------------------------------------- workload --

void check_domain(int32_t nx, int32_t ny, int32_t nz, int32_t fields) {
  if (nx < 1 || ny < 1 || nz < 1 || fields < 0)
    throw ValidationError("domain dimensions must be >= 1 (fields >= 0)");
}

std::vector<std::pair<int32_t, int32_t>> split_extent(int32_t extent, int32_t pieces) {
  std::vector<std::pair<int32_t, int32_t>> r(pieces);
  const int32_t q = extent / pieces, extra = extent % pieces;
  int32_t lo = 0;
  for (int32_t i = 0; i < pieces; ++i) {
    const int32_t hi = lo + q + (i < extra);
    r[i] = {lo, hi};
    lo = hi;
  }
  return r;
}

std::vector<Sub> strips_1d(int32_t nx, int32_t ny, int32_t k) {
  check_domain(nx, ny, 1, 0);
  if (k < 1 || k > ny) throw ValidationError("1d decomposition: k must be in [1, ny]");
  const auto rows = split_extent(ny, k);
  std::vector<Sub> out(k);
  for (int32_t i = 0; i < k; ++i) {
    Sub& s = out[i];
    s.vp = i;
    s.x0 = 0;
    s.x1 = nx;
    s.y0 = rows[i].first;
    s.y1 = rows[i].second;
    s.boundary = int64_t((i > 0) + (i + 1 < k)) * nx;
  }
  return out;
}

std::vector<Sub> tiles_2d(int32_t nx, int32_t ny, int32_t kx, int32_t ky) {
  check_domain(nx, ny, 1, 0);
  if (kx < 1 || kx > nx || ky < 1 || ky > ny)
    throw ValidationError("2d decomposition: tile counts exceed domain");
  const auto cols = split_extent(nx, kx), rows = split_extent(ny, ky);
  std::vector<Sub> out;
  out.reserve(size_t(kx) * ky);
  for (int32_t j = 0; j < ky; ++j)
    for (int32_t i = 0; i < kx; ++i) {
      Sub s;
      s.vp = j * kx + i;
      s.x0 = cols[i].first;
      s.x1 = cols[i].second;
      s.y0 = rows[j].first;
      s.y1 = rows[j].second;
      const int64_t w = s.x1 - s.x0, h = s.y1 - s.y0;
      s.boundary = h * ((i > 0) + (i + 1 < kx)) + w * ((j > 0) + (j + 1 < ky));
      out.push_back(s);
    }
  return out;
}

double Field2D::mean_over(const Sub& s) const {
  double acc = 0;
  for (int32_t y = s.y0; y < s.y1; ++y) {
    const double* row = c.data() + size_t(y) * nx;
    for (int32_t x = s.x0; x < s.x1; ++x) acc += row[x];
  }
  const int64_t n = s.cells();
  return n > 0 ? acc / double(n) : 0.0;
}

Field2D make_load_field(int32_t nx, int32_t ny, Pattern p, double heavy, double light,
                        const std::vector<Sub>& node0_subs) {
  check_domain(nx, ny, 1, 0);
  if (!(light >= 1.0) || !(heavy >= light))
    throw ValidationError("load field requires heavy_value >= light_value >= 1");
  Field2D f;
  f.nx = nx;
  f.ny = ny;
  f.c.assign(size_t(nx) * ny, light);
  if (p == kUpperHalfHeavy) {
    std::fill(f.c.begin(), f.c.begin() + size_t(ny / 2) * nx, heavy);
  } else if (p == kStaticNode0) {
    for (const Sub& s : node0_subs)
      for (int32_t y = s.y0; y < s.y1; ++y)
        std::fill(f.c.begin() + size_t(y) * nx + s.x0, f.c.begin() + size_t(y) * nx + s.x1,
                  heavy);
  } else if (p != kUniform) {
    throw ValidationError("unknown load pattern");
  }
  return f;
}

Field2D shift_rows_down(const Field2D& c, int32_t shift) {
  if (shift < 0 || shift > c.ny) throw ValidationError("advection shift must be in [0, ny]");
  if (shift == 0 || shift == c.ny) return c;
  Field2D o;
  o.nx = c.nx;
  o.ny = c.ny;
  o.c.resize(c.c.size());
  // row y of the output is row (y - shift) mod ny of the input
  const size_t row_bytes = size_t(c.nx);
  for (int32_t y = 0; y < c.ny; ++y) {
    const int32_t src = (y + c.ny - shift) % c.ny;
    std::copy_n(c.c.begin() + size_t(src) * row_bytes, row_bytes,
                o.c.begin() + size_t(y) * row_bytes);
  }
  return o;
}

Work physics_trips(const Sub& s, const Field2D& c, int32_t mzp) {
  const int64_t n = s.cells();
  if (n == 0) return {0, 0};
  const double mc = c.mean_over(s);
  return {double(n), mzp * mc - 1.0};
}

Work jacobi_items(const Sub& s, int32_t nz, int32_t fields) {
  const double items = double(s.cells()) * nz * fields;
  return {items, items > 0 ? 1.0 : 0.0};
}

int64_t halo_footprint(const Sub& s, int32_t nz, int32_t fields) {
  return s.boundary * nz * fields * int64_t(8);
}

int64_t chunk_footprint(const Sub& s, int32_t nz, int32_t fields) {
  return s.cells() * nz * fields * int64_t(8);
}

// ----------------------------------------------------------------- cluster --

std::vector<int32_t> block_mapping(int32_t K, int32_t P) {
  if (P < 1) throw ValidationError("proc count must be >= 1");
  if (K < P) throw ValidationError("vp count must be >= proc count");
  std::vector<int32_t> m(K);
  const int32_t q = K / P, extra = K % P;
  int32_t v = 0;
  for (int32_t p = 0; p < P; ++p)
    for (int32_t n = q + (p < extra); n > 0; --n) m[v++] = p;
  return m;
}

std::vector<int32_t> apply_moves(const std::vector<int32_t>& map, int32_t P,
                                 const std::vector<MoveRec>& moves) {
  std::vector<int32_t> out = map;
  const int32_t K = int32_t(map.size());
  for (const MoveRec& m : moves) {
    if (m.vp < 0 || m.vp >= K) throw ValidationError("move names an unknown vp");
    if (out[m.vp] != m.from)
      throw RuntimeFault("stale move: vp " + std::to_string(m.vp) + " is not on processor " +
                         std::to_string(m.from));
    if (m.to < 0 || m.to >= P) throw ValidationError("processor id out of range");
    out[m.vp] = m.to;
  }
  return out;
}

std::vector<double> totals_per_proc(const std::vector<double>& loads,
                                    const std::vector<int32_t>& map, int32_t P) {
  if (loads.size() != map.size())
    throw ValidationError("load vector length does not match vp count");
  std::vector<double> t(P, 0.0);
  for (size_t v = 0; v < map.size(); ++v) {
    if (map[v] < 0 || map[v] >= P) throw ValidationError("processor id out of range");
    t[map[v]] += loads[v];
  }
  return t;
}

double max_over_mean(const std::vector<double>& totals) {
  if (totals.empty()) throw ValidationError("no processor totals");
  double sum = 0.0, hi = totals[0];
  for (double t : totals) sum += t;
  if (sum <= 0.0) return 1.0;
  for (double t : totals) hi = hi < t ? t : hi;
  return hi / (sum / double(totals.size()));
}

// ---------------------------------------------------------------- balancer --

bool balance_needed(const std::vector<double>& totals, double threshold) {
  return max_over_mean(totals) > threshold;
}

std::vector<MoveRec> plan_greedy(const std::vector<double>& loads,
                                 const std::vector<int32_t>& map, int32_t P) {
  const int32_t K = int32_t(map.size());
  if (int32_t(loads.size()) != K) throw ValidationError("greedy_lb: load vector length mismatch");
  if (P < 1) throw ValidationError("proc count must be >= 1");
  // heaviest first; equal loads keep ascending vp order
  std::vector<int32_t> order(K);
  for (int32_t v = 0; v < K; ++v) order[v] = v;
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return loads[a] > loads[b] || (!(loads[b] > loads[a]) && !(loads[a] > loads[b]) && a < b);
  });
  std::vector<double> bin(P, 0.0);
  std::vector<int32_t> dest(K, 0);
  for (int32_t v : order) {
    // least-loaded processor, lowest id on ties
    const int32_t p = int32_t(std::min_element(bin.begin(), bin.end()) - bin.begin());
    dest[v] = p;
    bin[p] += loads[v];
  }
  std::vector<MoveRec> plan;
  for (int32_t v = 0; v < K; ++v)
    if (dest[v] != map[v]) plan.push_back({v, map[v], dest[v]});
  return plan;
}

namespace {
inline double larger(double a, double b) { return a < b ? b : a; }
}  // namespace

std::vector<MoveRec> plan_refine_swap(const std::vector<double>& loads,
                                      const std::vector<int32_t>& map, int32_t P,
                                      double tol) {
  const int32_t K = int32_t(map.size());
  if (int32_t(loads.size()) != K)
    throw ValidationError("refine_swap_lb: load vector length mismatch");
  if (tol < 0) throw ValidationError("refine_swap_lb: tolerance must be >= 0");
  if (P < 1) throw ValidationError("proc count must be >= 1");

  std::vector<int32_t> where = map;
  std::vector<double> acc = totals_per_proc(loads, where, P);
  double sum = 0.0;
  for (double a : acc) sum += a;
  const double avg = sum / P;
  const double ceil_load = avg * (1.0 + tol);

  std::vector<MoveRec> plan;
  std::vector<int32_t> donors, takers;
  auto members = [&](int32_t p, std::vector<int32_t>& out) {
    out.clear();
    for (int32_t v = 0; v < K; ++v)
      if (where[v] == p) out.push_back(v);
  };

  const int32_t max_rounds = K * P;
  for (int32_t round = 0; round < max_rounds; ++round) {
    int32_t hot = -1;
    for (int32_t p = 0; p < P; ++p)
      if (acc[p] > ceil_load && (hot < 0 || acc[p] > acc[hot])) hot = p;
    if (hot < 0) break;
    const double excess = acc[hot] - avg;
    members(hot, donors);

    // 1) single object from the hottest processor to an under-average one
    int32_t mv = -1, mq = -1;
    double mscore = 0;
    for (int32_t v : donors)
      for (int32_t q = 0; q < P; ++q) {
        if (q == hot || acc[q] >= avg) continue;
        const double after_src = acc[hot] - loads[v];
        const double after_dst = acc[q] + loads[v];
        const double ds = std::fabs(after_src - avg);
        if (ds >= excess || after_dst > ceil_load) continue;
        const double score = larger(ds, std::fabs(after_dst - avg));
        if (mv < 0 || score < mscore) { mv = v; mq = q; mscore = score; }
      }
    if (mv >= 0) {
      plan.push_back({mv, hot, mq});
      acc[hot] -= loads[mv];
      acc[mq] += loads[mv];
      where[mv] = mq;
      continue;
    }

    // 2) otherwise exchange one object each way with an under-average processor
    int32_t sa = -1, sb = -1, sq = -1;
    double sscore = 0;
    for (int32_t q = 0; q < P; ++q) {
      if (q == hot || acc[q] >= avg) continue;
      members(q, takers);
      for (int32_t a : donors)
        for (int32_t b : takers) {
          const double d = loads[a] - loads[b];
          if (d <= 0) continue;
          const double after_src = acc[hot] - d;
          const double after_dst = acc[q] + d;
          const double ds = std::fabs(after_src - avg);
          if (ds >= excess || after_dst > ceil_load) continue;
          const double score = larger(ds, std::fabs(after_dst - avg));
          if (sa < 0 || score < sscore) { sa = a; sb = b; sq = q; sscore = score; }
        }
    }
    if (sa < 0) break;
    plan.push_back({sa, hot, sq});
    plan.push_back({sb, sq, hot});
    const double d = loads[sa] - loads[sb];
    acc[hot] -= d;
    acc[sq] += d;
    where[sa] = sq;
    where[sb] = hot;
  }
  return plan;
}

// B200 extension (off-parity, opt-in Strategy 2): RefineSwapLB that keeps
// neighbouring chunks together.  Same rounds, thresholds and acceptance tests
// as plan_refine_swap, but among the admissible actions it takes the one that
// adds the fewest chunk faces between different processors (every such face is
// a halo strip over NVLink each step), the balance score breaking ties.
std::vector<MoveRec> plan_refine_adjacent(const std::vector<double>& loads,
                                          const std::vector<int32_t>& map, int32_t P, double tol,
                                          int32_t kind, int32_t kx, int32_t ky) {
  const int32_t K = int32_t(map.size());
  if (int32_t(loads.size()) != K)
    throw ValidationError("refine_adjacent_lb: load vector length mismatch");
  if (tol < 0) throw ValidationError("refine_adjacent_lb: tolerance must be >= 0");
  if (P < 1) throw ValidationError("proc count must be >= 1");
  if (kx < 1 || ky < 1 || (kind == 1 && kx * ky != K) || (kind == 0 && ky != K))
    throw ValidationError("refine_adjacent_lb: decomposition does not match the vp count");

  std::vector<int32_t> where = map;
  std::vector<double> acc = totals_per_proc(loads, where, P);
  double sum = 0.0;
  for (double a : acc) sum += a;
  const double avg = sum / P;
  const double ceil_load = avg * (1.0 + tol);
  // faces of v that would separate it from its neighbours if it sat on proc q
  auto cut_at = [&](int32_t v, int32_t q) {
    int32_t n = 0;
    for (int32_t d = 0; d < 4; ++d) {
      const int32_t nb = chunk_neighbor(kind, kx, ky, v, d);
      if (nb >= 0 && where[nb] != q) ++n;
    }
    return n;
  };

  std::vector<MoveRec> plan;
  std::vector<int32_t> donors, takers;
  auto members = [&](int32_t p, std::vector<int32_t>& out) {
    out.clear();
    for (int32_t v = 0; v < K; ++v)
      if (where[v] == p) out.push_back(v);
  };
  const int32_t max_rounds = K * P;
  for (int32_t round = 0; round < max_rounds; ++round) {
    int32_t hot = -1;
    for (int32_t p = 0; p < P; ++p)
      if (acc[p] > ceil_load && (hot < 0 || acc[p] > acc[hot])) hot = p;
    if (hot < 0) break;
    const double excess = acc[hot] - avg;
    members(hot, donors);

    int32_t mv = -1, mq = -1, mcut = 0;
    double mscore = 0;
    for (int32_t v : donors)
      for (int32_t q = 0; q < P; ++q) {
        if (q == hot || acc[q] >= avg) continue;
        const double after_src = acc[hot] - loads[v];
        const double after_dst = acc[q] + loads[v];
        const double ds = std::fabs(after_src - avg);
        if (ds >= excess || after_dst > ceil_load) continue;
        const double score = larger(ds, std::fabs(after_dst - avg));
        const int32_t dcut = cut_at(v, q) - cut_at(v, hot);
        if (mv < 0 || dcut < mcut || (dcut == mcut && score < mscore)) {
          mv = v;
          mq = q;
          mscore = score;
          mcut = dcut;
        }
      }
    if (mv >= 0) {
      plan.push_back({mv, hot, mq});
      acc[hot] -= loads[mv];
      acc[mq] += loads[mv];
      where[mv] = mq;
      continue;
    }
    int32_t sa = -1, sb = -1, sq = -1, scut = 0;
    double sscore = 0;
    for (int32_t q = 0; q < P; ++q) {
      if (q == hot || acc[q] >= avg) continue;
      members(q, takers);
      for (int32_t a : donors)
        for (int32_t b : takers) {
          const double d = loads[a] - loads[b];
          if (d <= 0) continue;
          const double after_src = acc[hot] - d;
          const double after_dst = acc[q] + d;
          const double ds = std::fabs(after_src - avg);
          if (ds >= excess || after_dst > ceil_load) continue;
          const double score = larger(ds, std::fabs(after_dst - avg));
          // cut change of moving a to q, then b to hot
          int32_t dcut = cut_at(a, q) - cut_at(a, hot);
          where[a] = q;
          dcut += cut_at(b, hot) - cut_at(b, q);
          where[a] = hot;
          if (sa < 0 || dcut < scut || (dcut == scut && score < sscore)) {
            sa = a;
            sb = b;
            sq = q;
            sscore = score;
            scut = dcut;
          }
        }
    }
    if (sa < 0) break;
    plan.push_back({sa, hot, sq});
    plan.push_back({sb, sq, hot});
    const double d = loads[sa] - loads[sb];
    acc[hot] -= d;
    acc[sq] += d;
    where[sa] = sq;
    where[sb] = hot;
  }
  return plan;
}

// ------------------------------------------------- capacity-aware balancers --

void Capacity::validate(int32_t K, int32_t P) const {
  if (int32_t(vp_bytes.size()) != K) throw ValidationError("capacity: vp_bytes length mismatch");
  if (int32_t(bin_of_proc.size()) != P)
    throw ValidationError("capacity: bin_of_proc length mismatch");
  for (int64_t b : vp_bytes)
    if (b < 0) throw ValidationError("capacity: chunk bytes must be >= 0");
  for (int32_t b : bin_of_proc)
    if (b < 0 || b >= int32_t(bin_cap.size())) throw ValidationError("capacity: bin out of range");
  for (int64_t c : bin_cap)
    if (c < 0) throw ValidationError("capacity: bin capacity must be >= 0");
}

std::vector<MoveRec> plan_greedy_capacity(const std::vector<double>& loads,
                                          const std::vector<int32_t>& map, int32_t P,
                                          const Capacity& cap) {
  const int32_t K = int32_t(map.size());
  if (int32_t(loads.size()) != K) throw ValidationError("greedy_lb: load vector length mismatch");
  if (P < 1) throw ValidationError("proc count must be >= 1");
  cap.validate(K, P);
  // plan_greedy's order and least-loaded rule, over the processors whose bin
  // still has room for the chunk
  std::vector<int32_t> order(K);
  for (int32_t v = 0; v < K; ++v) order[v] = v;
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return loads[a] > loads[b] || (!(loads[b] > loads[a]) && !(loads[a] > loads[b]) && a < b);
  });
  std::vector<double> bin(P, 0.0);
  std::vector<int64_t> used(cap.bin_cap.size(), 0);
  std::vector<int32_t> dest(K, 0);
  for (int32_t v : order) {
    int32_t p = -1;
    for (int32_t q = 0; q < P; ++q) {
      const int32_t b = cap.bin_of_proc[q];
      if (used[b] + cap.vp_bytes[v] > cap.bin_cap[b]) continue;
      if (p < 0 || bin[q] < bin[p]) p = q;
    }
    if (p < 0) {
      // no bin has room: the processor whose bin has the most room left
      for (int32_t q = 0; q < P; ++q) {
        const int32_t b = cap.bin_of_proc[q], bp = p < 0 ? -1 : cap.bin_of_proc[p];
        if (p < 0 || cap.bin_cap[b] - used[b] > cap.bin_cap[bp] - used[bp]) p = q;
      }
    }
    dest[v] = p;
    bin[p] += loads[v];
    used[cap.bin_of_proc[p]] += cap.vp_bytes[v];
  }
  // Repair (only when the greedy pass had to overfill): a bin over capacity
  // holds at least one chunk that moved in (its own chunks fitted before the
  // plan), so return moved-in chunks home, lightest first, until every bin
  // fits; each return shrinks the plan, so this ends at the latest with the
  // starting layout.
  for (bool over = true; over;) {
    over = false;
    for (size_t b = 0; b < used.size(); ++b) {
      while (used[b] > cap.bin_cap[b]) {
        int32_t back = -1;
        for (int32_t v = 0; v < K; ++v)
          if (dest[v] != map[v] && cap.bin_of_proc[dest[v]] == int32_t(b) &&
              cap.bin_of_proc[map[v]] != int32_t(b) &&
              (back < 0 || loads[v] < loads[back] || (loads[v] == loads[back] && v < back)))
            back = v;
        if (back < 0) break;  // the bin was over capacity before the plan
        used[b] -= cap.vp_bytes[back];
        used[cap.bin_of_proc[map[back]]] += cap.vp_bytes[back];
        dest[back] = map[back];
        over = true;
      }
    }
  }
  std::vector<MoveRec> plan;
  for (int32_t v = 0; v < K; ++v)
    if (dest[v] != map[v]) plan.push_back({v, map[v], dest[v]});
  return plan;
}

std::vector<MoveRec> plan_refine_capacity(const std::vector<double>& loads,
                                          const std::vector<int32_t>& map, int32_t P, double tol,
                                          const Capacity& cap) {
  const int32_t K = int32_t(map.size());
  if (int32_t(loads.size()) != K)
    throw ValidationError("refine_swap_lb: load vector length mismatch");
  if (tol < 0) throw ValidationError("refine_swap_lb: tolerance must be >= 0");
  if (P < 1) throw ValidationError("proc count must be >= 1");
  cap.validate(K, P);
  std::vector<int32_t> where = map;
  std::vector<double> acc = totals_per_proc(loads, where, P);
  std::vector<int64_t> used(cap.bin_cap.size(), 0);
  for (int32_t v = 0; v < K; ++v) used[cap.bin_of_proc[where[v]]] += cap.vp_bytes[v];
  // a bin may take `delta` more bytes if it shrinks or stays within capacity
  auto fits = [&](int32_t b, int64_t delta) { return delta <= 0 || used[b] + delta <= cap.bin_cap[b]; };
  double sum = 0.0;
  for (double a : acc) sum += a;
  const double avg = sum / P;
  const double ceil_load = avg * (1.0 + tol);

  std::vector<MoveRec> plan;
  std::vector<int32_t> donors, takers;
  auto members = [&](int32_t p, std::vector<int32_t>& out) {
    out.clear();
    for (int32_t v = 0; v < K; ++v)
      if (where[v] == p) out.push_back(v);
  };
  const int32_t max_rounds = K * P;
  for (int32_t round = 0; round < max_rounds; ++round) {
    int32_t hot = -1;
    for (int32_t p = 0; p < P; ++p)
      if (acc[p] > ceil_load && (hot < 0 || acc[p] > acc[hot])) hot = p;
    if (hot < 0) break;
    const double excess = acc[hot] - avg;
    const int32_t bh = cap.bin_of_proc[hot];
    members(hot, donors);
    int32_t mv = -1, mq = -1;
    double mscore = 0;
    for (int32_t v : donors)
      for (int32_t q = 0; q < P; ++q) {
        if (q == hot || acc[q] >= avg) continue;
        const double after_src = acc[hot] - loads[v];
        const double after_dst = acc[q] + loads[v];
        const double ds = std::fabs(after_src - avg);
        if (ds >= excess || after_dst > ceil_load) continue;
        const int32_t bq = cap.bin_of_proc[q];
        if (bq != bh && !fits(bq, cap.vp_bytes[v])) continue;
        const double score = larger(ds, std::fabs(after_dst - avg));
        if (mv < 0 || score < mscore) { mv = v; mq = q; mscore = score; }
      }
    if (mv >= 0) {
      plan.push_back({mv, hot, mq});
      acc[hot] -= loads[mv];
      acc[mq] += loads[mv];
      const int32_t bq = cap.bin_of_proc[mq];
      used[bh] -= cap.vp_bytes[mv];
      used[bq] += cap.vp_bytes[mv];
      where[mv] = mq;
      continue;
    }
    int32_t sa = -1, sb = -1, sq = -1;
    double sscore = 0;
    for (int32_t q = 0; q < P; ++q) {
      if (q == hot || acc[q] >= avg) continue;
      const int32_t bq = cap.bin_of_proc[q];
      members(q, takers);
      for (int32_t a : donors)
        for (int32_t b : takers) {
          const double d = loads[a] - loads[b];
          if (d <= 0) continue;
          const double after_src = acc[hot] - d;
          const double after_dst = acc[q] + d;
          const double ds = std::fabs(after_src - avg);
          if (ds >= excess || after_dst > ceil_load) continue;
          if (bq != bh) {
            const int64_t db = cap.vp_bytes[a] - cap.vp_bytes[b];
            if (!fits(bq, db) || !fits(bh, -db)) continue;
          }
          const double score = larger(ds, std::fabs(after_dst - avg));
          if (sa < 0 || score < sscore) { sa = a; sb = b; sq = q; sscore = score; }
        }
    }
    if (sa < 0) break;
    plan.push_back({sa, hot, sq});
    plan.push_back({sb, sq, hot});
    const double d = loads[sa] - loads[sb];
    acc[hot] -= d;
    acc[sq] += d;
    const int64_t db = cap.vp_bytes[sa] - cap.vp_bytes[sb];
    used[cap.bin_of_proc[sq]] += db;
    used[bh] -= db;
    where[sa] = sq;
    where[sb] = hot;
  }
  return plan;
}

// ------------------------------------------------------------ modelled costs --

void GpuCostModel::validate() const {
  if (launch_overhead < 0 || per_item_time < 0 || saturation_floor < 0)
    throw ValidationError("gpu model times must be >= 0");
  if (h2d_bandwidth <= 0 || d2h_bandwidth <= 0)
    throw ValidationError("gpu model bandwidths must be > 0");
  if (async_overlap_gain < 0 || async_overlap_gain >= 1)
    throw ValidationError("gpu model async_overlap_gain must be in [0, 1)");
}

double kernel_time_sync_model(const Work& w, const GpuCostModel& g) {
  if (w.total() <= 0) return 0.0;
  const double t = g.launch_overhead + g.per_item_time * w.total();
  return g.saturation_floor < t ? t : g.saturation_floor;
}

double transfer_time_model(double bytes, bool host_to_device, const GpuCostModel& g) {
  if (bytes < 0) throw ValidationError("transfer bytes must be >= 0");
  if (bytes == 0) return 0.0;
  return bytes / (host_to_device ? g.h2d_bandwidth : g.d2h_bandwidth);
}

double node_gpu_schedule_model(const std::vector<double>& jobs, int32_t mode,
                               const GpuCostModel& g) {
  double sum = 0.0, mx = 0.0;
  for (double j : jobs) {
    if (j < 0) throw ValidationError("kernel durations must be >= 0");
    sum += j;
    mx = mx < j ? j : mx;
  }
  if (mode == kSync || jobs.size() <= 1) return sum;
  const double overlapped = sum * (1.0 - g.async_overlap_gain);
  return overlapped < mx ? mx : overlapped;
}

double plan_cost_model(const std::vector<MoveRec>& plan, const std::vector<int64_t>& data_bytes,
                       int32_t procs_per_node, int32_t nodes, double net_bandwidth,
                       double net_latency, const GpuCostModel& g) {
  if (procs_per_node < 1 || nodes < 1) throw ValidationError("cluster counts must be >= 1");
  std::vector<double> per_node(nodes, 0.0);
  for (const MoveRec& m : plan) {
    if (m.vp < 0 || m.vp >= int32_t(data_bytes.size()))
      throw ValidationError("move names an unknown vp");
    const double bytes = double(data_bytes[m.vp]);
    const int32_t a = m.from / procs_per_node, b = m.to / procs_per_node;
    if (a < 0 || a >= nodes || b < 0 || b >= nodes) throw ValidationError("processor id out of range");
    per_node[a] += transfer_time_model(bytes, false, g);
    per_node[b] += transfer_time_model(bytes, true, g);
    if (a != b) {
      const double hop = bytes / net_bandwidth + net_latency;
      per_node[a] += hop;
      per_node[b] += hop;
    }
  }
  double mx = 0.0;
  for (double c : per_node) mx = mx < c ? c : mx;
  return per_node.empty() ? 0.0 : mx;
}

// ------------------------------------------------------------ epoch policy --

Decision decide_epoch(const std::vector<double>& loads, const std::vector<int32_t>& map,
                      int32_t P, int32_t epoch, int32_t epochs, int32_t& balance_calls,
                      int32_t first_strategy, int32_t later_strategy, double threshold,
                      double tolerance, int32_t kind, int32_t kx, int32_t ky,
                      const Capacity* cap) {
  Decision d;
  d.totals = totals_per_proc(loads, map, P);
  d.imbalance_before = max_over_mean(d.totals);
  d.imbalance_after = d.imbalance_before;
  if (epoch < epochs && balance_needed(d.totals, threshold)) {
    d.strategy = balance_calls == 0 ? first_strategy : later_strategy;
    if (d.strategy == kGreedy)
      d.plan = cap ? plan_greedy_capacity(loads, map, P, *cap) : plan_greedy(loads, map, P);
    else if (d.strategy == kRefineAdjacent) {
      if (kind < 0) throw ValidationError("strategy 2 (refine_adjacent) needs the decomposition");
      d.plan = plan_refine_adjacent(loads, map, P, tolerance, kind, kx, ky);
    } else
      d.plan = cap ? plan_refine_capacity(loads, map, P, tolerance, *cap)
                   : plan_refine_swap(loads, map, P, tolerance);
    ++balance_calls;
    if (!d.plan.empty())
      d.imbalance_after = max_over_mean(totals_per_proc(loads, apply_moves(map, P, d.plan), P));
  }
  return d;
}

// -------------------------------------------------------- exchange schedule --

int32_t chunk_neighbor(int32_t kind, int32_t kx, int32_t ky, int32_t vp, int32_t side) {
  if (kind == 0) kx = 1;  // strips: vertical neighbours only
  const int32_t i = vp % kx, j = vp / kx;
  switch (side) {
    case 0: return i > 0 ? vp - 1 : -1;
    case 1: return i + 1 < kx ? vp + 1 : -1;
    case 2: return j > 0 ? vp - kx : -1;
    default: return j + 1 < ky ? vp + kx : -1;
  }
}

void exchange_schedule(const std::vector<Sub>& subs, int32_t kind, int32_t kx, int32_t ky,
                       const std::vector<int32_t>& rank_of_vp, int32_t world, int32_t rank,
                       int64_t per_cell, std::vector<FaceXfer>& sends,
                       std::vector<FaceXfer>& recvs) {
  sends.clear();
  recvs.clear();
  const int32_t K = int32_t(subs.size());
  int64_t soff = 0, roff = 0;
  for (int32_t q = 0; q < world; ++q) {
    if (q == rank) continue;
    // strips this rank sends to q: my chunk v, face d bordering a chunk on q
    for (int32_t v = 0; v < K; ++v) {
      if (rank_of_vp[v] != rank) continue;
      for (int32_t d = 0; d < 4; ++d) {
        const int32_t n = chunk_neighbor(kind, kx, ky, v, d);
        if (n < 0 || rank_of_vp[n] != q) continue;
        const int32_t len = d < 2 ? subs[v].h() : subs[v].w();
        const int32_t lenp = (len + 1) & ~1;
        sends.push_back({q, v, d, n, len, lenp, soff});
        soff += per_cell * lenp;
      }
    }
    // strips q sends to this rank, in q's (sender vp, side) order
    for (int32_t v = 0; v < K; ++v) {
      if (rank_of_vp[v] != q) continue;
      for (int32_t d = 0; d < 4; ++d) {
        const int32_t n = chunk_neighbor(kind, kx, ky, v, d);
        if (n < 0 || rank_of_vp[n] != rank) continue;
        const int32_t len = d < 2 ? subs[v].h() : subs[v].w();
        const int32_t lenp = (len + 1) & ~1;
        recvs.push_back({q, v, d, n, len, lenp, roff});
        roff += per_cell * lenp;
      }
    }
  }
}

// ------------------------------------------------------------- measurement --

SampleStore::SampleStore(int32_t K, int32_t async_steps, int32_t sync_steps)
    : K_(K), async_(async_steps), sync_(sync_steps) {
  if (K < 0) throw ValidationError("vp count must be >= 0");
  if (async_steps < 0) throw ValidationError("window.async_steps must be >= 0");
  if (sync_steps < 1) throw ValidationError("window.sync_steps must be >= 1");
  seen_.assign(size_t(K) * (async_ + sync_), 0);
}

void SampleStore::add(int32_t vp, int32_t step, int32_t mode, double value) {
  if (vp < 0 || vp >= K_) throw ValidationError("sample vp out of range");
  if (step < 0 || step >= async_ + sync_)
    throw RuntimeFault("sample step outside the current epoch");
  if (value < 0) throw ValidationError("sample value must be >= 0");
  uint8_t& slot = seen_[size_t(vp) * (async_ + sync_) + step];
  if (slot)
    throw RuntimeFault("duplicate sample for vp " + std::to_string(vp) + " step " +
                       std::to_string(step));
  slot = 1;
  rec_.push_back({vp, step, mode, value});
}

void SampleStore::reset() {
  rec_.clear();
  std::fill(seen_.begin(), seen_.end(), 0);
}

std::vector<double> SampleStore::sync_means() const {
  std::vector<double> s(K_, 0.0);
  std::vector<int32_t> n(K_, 0);
  for (const Rec& r : rec_)
    if (r.mode == kSync) {
      s[r.vp] += r.v;
      ++n[r.vp];
    }
  for (int32_t v = 0; v < K_; ++v) {
    if (n[v] == 0)
      throw RuntimeFault("incomplete measurement: vp " + std::to_string(v) +
                         " has no synchronous sample in this epoch");
    s[v] = s[v] / n[v];
  }
  return s;
}

double plan_cost_nvlink_model(const std::vector<MoveRec>& plan,
                              const std::vector<int64_t>& data_bytes, int32_t procs_per_gpu,
                              int32_t gpus, double link_bandwidth, double latency) {
  if (procs_per_gpu < 1 || gpus < 1) throw ValidationError("cluster sizes must be >= 1");
  if (link_bandwidth <= 0) throw ValidationError("link bandwidth must be > 0");
  if (latency < 0) throw ValidationError("link latency must be >= 0");
  std::vector<double> out_b(gpus, 0.0), in_b(gpus, 0.0);
  std::vector<int32_t> count(gpus, 0);
  for (const MoveRec& m : plan) {
    if (m.vp < 0 || m.vp >= int32_t(data_bytes.size()))
      throw ValidationError("move vp out of range");
    const int32_t a = m.from / procs_per_gpu, b = m.to / procs_per_gpu;
    if (m.from < 0 || m.to < 0 || a >= gpus || b >= gpus)
      throw ValidationError("move processor out of range");
    if (a == b) continue;
    out_b[a] += double(data_bytes[m.vp]);
    in_b[b] += double(data_bytes[m.vp]);
    ++count[a];
    ++count[b];
  }
  double worst = 0.0;
  for (int32_t g = 0; g < gpus; ++g) {
    const double t = (out_b[g] > in_b[g] ? out_b[g] : in_b[g]) / link_bandwidth +
                     latency * count[g];
    if (t > worst) worst = t;
  }
  return worst;
}

// ---- calibration --------------------------------------------------------------
namespace {

// squared relative error of max(floor, launch + rate * total) over the samples
// (gpu_cost.hpp:94-104); out-of-domain parameters are rejected with a huge value
double hinge_error(const std::vector<CalibSample>& ss, const std::array<double, 3>& p) {
  const double launch = p[0], rate = p[1], floor = p[2];
  if (launch < 0 || rate <= 0 || floor < 0) return 1e30;
  double e = 0.0;
  for (const CalibSample& s : ss) {
    const double line = launch + rate * s.w.total();
    const double pred = floor < line ? line : floor;
    const double rel = (pred - s.seconds) / s.seconds;
    e += rel * rel;
  }
  return e;
}

// Nelder-Mead on (launch, rate, floor) from `start` (gpu_cost.hpp:108-168):
// initial simplex = start plus each coordinate scaled by 1.25 (1e-6 if zero);
// reflect 1, expand 2, contract +-0.5, shrink 0.5 toward the best; at most
// 2000 iterations, stop when the spread of values is below 1e-16 (1 + best)
std::array<double, 3> nelder_mead(const std::vector<CalibSample>& ss, std::array<double, 3> start) {
  using Pt = std::array<double, 3>;
  std::array<Pt, 4> x;
  std::array<double, 4> fx;
  x[0] = start;
  for (int i = 0; i < 3; ++i) {
    x[i + 1] = start;
    x[i + 1][i] = start[i] != 0.0 ? start[i] * 1.25 : 1e-6;
  }
  for (int i = 0; i < 4; ++i) fx[i] = hinge_error(ss, x[i]);
  for (int it = 0; it < 2000; ++it) {
    // exchange ordering by value (ties keep their relative order)
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j)
        if (fx[j] < fx[i]) {
          std::swap(fx[i], fx[j]);
          std::swap(x[i], x[j]);
        }
    if (fx[3] - fx[0] < 1e-16 * (1.0 + fx[0])) break;
    Pt c{0.0, 0.0, 0.0};
    for (int i = 0; i < 3; ++i)
      for (int d = 0; d < 3; ++d) c[d] += x[i][d] / 3.0;
    auto along = [&](double t) {
      Pt q;
      for (int d = 0; d < 3; ++d) q[d] = c[d] + t * (c[d] - x[3][d]);
      return q;
    };
    const Pt r = along(1.0);
    const double fr = hinge_error(ss, r);
    if (fr < fx[0]) {
      const Pt e = along(2.0);
      const double fe = hinge_error(ss, e);
      if (fe < fr) {
        x[3] = e;
        fx[3] = fe;
      } else {
        x[3] = r;
        fx[3] = fr;
      }
    } else if (fr < fx[2]) {
      x[3] = r;
      fx[3] = fr;
    } else {
      const Pt k = along(fr < fx[3] ? 0.5 : -0.5);
      const double fk = hinge_error(ss, k);
      if (fk < (fr < fx[3] ? fr : fx[3])) {
        x[3] = k;
        fx[3] = fk;
      } else {
        for (int i = 1; i < 4; ++i) {
          for (int d = 0; d < 3; ++d) x[i][d] = 0.5 * (x[i][d] + x[0][d]);
          fx[i] = hinge_error(ss, x[i]);
        }
      }
    }
  }
  int best = 0;
  for (int i = 1; i < 4; ++i)
    if (fx[i] < fx[best]) best = i;
  return x[best];
}

// ordinary least squares y = a + b x (gpu_cost.hpp:171-181)
std::pair<double, double> line_fit(const std::vector<std::pair<double, double>>& xy) {
  const double n = double(xy.size());
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  for (const auto& p : xy) {
    sx += p.first;
    sy += p.second;
    sxx += p.first * p.first;
    sxy += p.first * p.second;
  }
  const double den = n * sxx - sx * sx;
  if (den == 0) throw ValidationError("degenerate calibration samples (identical work)");
  const double b = (n * sxy - sx * sy) / den;
  return {(sy - b * sx) / n, b};
}

}  // namespace

GpuFit calibrate_gpu_model(const std::vector<CalibSample>& ss, const GpuCostModel& defaults) {
  if (ss.size() < 3) throw ValidationError("gpu calibration needs >= 3 samples");
  for (const CalibSample& s : ss)
    if (s.seconds <= 0 || s.w.total() <= 0)
      throw ValidationError("gpu calibration samples must have positive work and time");
  double tmin = ss[0].seconds;
  for (const CalibSample& s : ss)
    if (s.seconds < tmin) tmin = s.seconds;
  std::vector<std::pair<double, double>> above;
  int floor_rows = 0;
  for (const CalibSample& s : ss) {
    if (s.seconds <= tmin * 1.10)
      ++floor_rows;
    else
      above.emplace_back(s.w.total(), s.seconds);
  }
  std::array<double, 3> p{0.0, 0.0, 0.0};  // launch, rate, floor
  if (above.size() >= 2) {
    const auto ab = line_fit(above);
    p = {ab.first > 0.0 ? ab.first : 0.0, ab.second, floor_rows >= 1 ? tmin : 0.0};
  } else {
    std::vector<std::pair<double, double>> all;
    for (const CalibSample& s : ss) all.emplace_back(s.w.total(), s.seconds);
    const auto ab = line_fit(all);
    p = {ab.first > 0.0 ? ab.first : 0.0, ab.second, 0.0};
  }
  if (p[1] <= 0) throw ValidationError("gpu calibration produced a non-positive rate");
  const double e0 = hinge_error(ss, p);
  if (e0 > 1e-12) {
    const double f0 = p[2] > tmin * 0.5 ? p[2] : tmin * 0.5;
    const std::array<double, 3> q = nelder_mead(ss, {p[0], p[1], f0});
    if (hinge_error(ss, q) < e0) p = q;
  }
  GpuFit out;
  out.model = defaults;
  out.model.launch_overhead = p[0];
  out.model.per_item_time = p[1];
  out.model.saturation_floor = p[2];
  out.model.validate();
  for (const CalibSample& s : ss) {
    const double r = std::abs(kernel_time_sync_model(s.w, out.model) - s.seconds) / s.seconds;
    if (r > out.max_rel_residual) out.max_rel_residual = r;
  }
  return out;
}

double calibrate_cpu_model(const std::vector<CalibSample>& ss) {
  if (ss.empty()) throw ValidationError("cpu calibration needs samples");
  double sxx = 0, sxy = 0;
  for (const CalibSample& s : ss) {
    const double x = s.w.total();
    sxx += x * x;
    sxy += x * s.seconds;
  }
  if (sxx == 0) throw ValidationError("degenerate cpu calibration samples");
  const double r = sxy / sxx;
  if (r <= 0) throw ValidationError("cpu model per_item_time must be > 0");
  return r;
}

double cpu_time_model(const Work& w, double cpu_per_item) { return cpu_per_item * w.total(); }

void scaling_probe_model(int32_t n, const std::vector<int32_t>& m_list, double inner,
                         const GpuCostModel& g, double cpu_per_item, std::vector<double>& cpu_s,
                         std::vector<double>& gpu_s) {
  if (m_list.empty()) throw ValidationError("scaling probe needs at least one M");
  cpu_s.clear();
  gpu_s.clear();
  for (int32_t m : m_list) {
    const Work w{double(n - 2) * (m - 2), inner};
    cpu_s.push_back(cpu_time_model(w, cpu_per_item));
    gpu_s.push_back(kernel_time_sync_model(w, g));
  }
}

}  // namespace odb
