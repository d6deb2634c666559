// extern "C" surface of include/overdeck_b200.h for the pure host model.
// Exceptions never cross the boundary: ValidationError -> 2, RuntimeFault and
// any other failure -> 3, message kept per thread for od_last_error().
#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "../../include/overdeck_b200.h"
#include "od_capi_util.hpp"
#include "od_model.hpp"

namespace odb {
thread_local std::string g_last_error;

int fail_with(const std::exception& e, int code) {
  g_last_error = e.what();
  return code;
}
}  // namespace odb

using namespace odb;

namespace {

Sub to_sub(const od_subdomain& s) {
  Sub r;
  r.vp = s.owner_vp;
  r.x0 = s.x_begin;
  r.x1 = s.x_end;
  r.y0 = s.y_begin;
  r.y1 = s.y_end;
  r.boundary = s.boundary_cells;
  return r;
}

void put_subs(const std::vector<Sub>& v, od_subdomain* out) {
  for (size_t i = 0; i < v.size(); ++i)
    out[i] = od_subdomain{v[i].vp, v[i].x0, v[i].x1, v[i].y0, v[i].y1, v[i].boundary};
}

void need(const void* p, const char* what) {
  if (!p) throw ValidationError(std::string("null pointer: ") + what);
}

Field2D field_view(const double* c, int32_t nx, int32_t ny) {
  check_domain(nx, ny, 1, 0);
  need(c, "load field");
  Field2D f;
  f.nx = nx;
  f.ny = ny;
  f.c.assign(c, c + size_t(nx) * ny);
  return f;
}

void check_sub_in(const od_subdomain* s, int32_t nx, int32_t ny) {
  need(s, "subdomain");
  if (s->x_begin < 0 || s->x_end > nx || s->x_begin > s->x_end || s->y_begin < 0 ||
      s->y_end > ny || s->y_begin > s->y_end)
    throw ValidationError("subdomain outside the load field");
}

std::vector<int32_t> map_view(const int32_t* map, int32_t K, int32_t P) {
  if (K < 0) throw ValidationError("vp count must be >= 0");
  if (P < 1) throw ValidationError("proc count must be >= 1");
  if (K > 0) need(map, "mapping");
  std::vector<int32_t> m(map, map + K);
  for (int32_t p : m)
    if (p < 0 || p >= P) throw ValidationError("processor id out of range");
  return m;
}

std::vector<double> vec_view(const double* a, int32_t n, const char* what) {
  if (n < 0) throw ValidationError(std::string("negative length: ") + what);
  if (n > 0) need(a, what);
  return std::vector<double>(a, a + n);
}

int emit_moves(const std::vector<MoveRec>& plan, od_move* out, int32_t cap, int32_t* n_out) {
  need(n_out, "n_out");
  *n_out = int32_t(plan.size());
  if (int32_t(plan.size()) > cap) throw ValidationError("move buffer too small");
  if (!plan.empty()) need(out, "out");
  for (size_t i = 0; i < plan.size(); ++i) out[i] = od_move{plan[i].vp, plan[i].from, plan[i].to};
  return OD_OK;
}

}  // namespace

extern "C" {

const char* od_last_error(void) { return g_last_error.c_str(); }
int32_t od_abi_version(void) { return 1; }

int od_decompose_1d(int32_t nx, int32_t ny, int32_t k, od_subdomain* out) {
  return guarded([&] {
    auto s = strips_1d(nx, ny, k);
    need(out, "out");
    put_subs(s, out);
  });
}

int od_decompose_2d(int32_t nx, int32_t ny, int32_t kx, int32_t ky, od_subdomain* out) {
  return guarded([&] {
    auto s = tiles_2d(nx, ny, kx, ky);
    need(out, "out");
    put_subs(s, out);
  });
}

int od_init_load_field(int32_t nx, int32_t ny, int32_t pattern, double heavy_value,
                       double light_value, const od_subdomain* node0_subs, int32_t n_node0,
                       double* out) {
  return guarded([&] {
    if (pattern < OD_UNIFORM || pattern > OD_UPPER_HALF_HEAVY)
      throw ValidationError("unknown load pattern");
    std::vector<Sub> subs;
    if (n_node0 > 0) need(node0_subs, "node0_subs");
    for (int32_t i = 0; i < n_node0; ++i) {
      check_sub_in(&node0_subs[i], nx, ny);
      subs.push_back(to_sub(node0_subs[i]));
    }
    Field2D f = make_load_field(nx, ny, Pattern(pattern), heavy_value, light_value, subs);
    need(out, "out");
    std::memcpy(out, f.c.data(), f.c.size() * sizeof(double));
  });
}

int od_advect_load_field(const double* c, int32_t nx, int32_t ny, int32_t shift_rows,
                         double* out) {
  return guarded([&] {
    Field2D f = shift_rows_down(field_view(c, nx, ny), shift_rows);
    need(out, "out");
    std::memcpy(out, f.c.data(), f.c.size() * sizeof(double));
  });
}

int od_mean_over(const double* c, int32_t nx, int32_t ny, const od_subdomain* sub,
                 double* out) {
  return guarded([&] {
    check_sub_in(sub, nx, ny);
    need(out, "out");
    *out = field_view(c, nx, ny).mean_over(to_sub(*sub));
  });
}

int od_physics_work(const od_subdomain* sub, const double* c, int32_t nx, int32_t ny,
                    int32_t mzp, od_kernel_work* out) {
  return guarded([&] {
    check_sub_in(sub, nx, ny);
    need(out, "out");
    Work w = physics_trips(to_sub(*sub), field_view(c, nx, ny), mzp);
    *out = od_kernel_work{w.items, w.depth};
  });
}

int od_jacobi_work(const od_subdomain* sub, int32_t nz, int32_t fields, od_kernel_work* out) {
  return guarded([&] {
    need(sub, "subdomain");
    need(out, "out");
    Work w = jacobi_items(to_sub(*sub), nz, fields);
    *out = od_kernel_work{w.items, w.depth};
  });
}

int od_halo_bytes(const od_subdomain* sub, int32_t nz, int32_t fields, int64_t* out) {
  return guarded([&] {
    need(sub, "subdomain");
    need(out, "out");
    *out = halo_footprint(to_sub(*sub), nz, fields);
  });
}

int od_subdomain_bytes(const od_subdomain* sub, int32_t nz, int32_t fields, int64_t* out) {
  return guarded([&] {
    need(sub, "subdomain");
    need(out, "out");
    *out = chunk_footprint(to_sub(*sub), nz, fields);
  });
}

int od_initial_block_mapping(int32_t vp_count, int32_t proc_count, int32_t* map) {
  return guarded([&] {
    auto m = block_mapping(vp_count, proc_count);
    if (vp_count > 0) need(map, "map");
    std::memcpy(map, m.data(), m.size() * sizeof(int32_t));
  });
}

int od_apply_plan(const int32_t* map_in, int32_t vp_count, int32_t proc_count,
                  const od_move* moves, int32_t n_moves, int32_t* map_out) {
  return guarded([&] {
    auto m = map_view(map_in, vp_count, proc_count);
    if (n_moves < 0) throw ValidationError("negative move count");
    if (n_moves > 0) need(moves, "moves");
    std::vector<MoveRec> mv(n_moves);
    for (int32_t i = 0; i < n_moves; ++i) mv[i] = {moves[i].vp, moves[i].from, moves[i].to};
    auto r = apply_moves(m, proc_count, mv);
    if (vp_count > 0) need(map_out, "map_out");
    std::memcpy(map_out, r.data(), r.size() * sizeof(int32_t));
  });
}

int od_proc_loads(const double* loads, int32_t n_loads, const int32_t* map, int32_t vp_count,
                  int32_t proc_count, double* totals) {
  return guarded([&] {
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    auto t = totals_per_proc(l, m, proc_count);
    need(totals, "totals");
    std::memcpy(totals, t.data(), t.size() * sizeof(double));
  });
}

int od_imbalance_ratio(const double* totals, int32_t n, double* out) {
  return guarded([&] {
    auto t = vec_view(totals, n, "totals");
    need(out, "out");
    *out = max_over_mean(t);
  });
}

int od_should_balance(const double* totals, int32_t n, double trigger_threshold, int32_t* out) {
  return guarded([&] {
    auto t = vec_view(totals, n, "totals");
    need(out, "out");
    *out = balance_needed(t, trigger_threshold) ? 1 : 0;
  });
}

int od_greedy_lb(const double* loads, int32_t n_loads, const int32_t* map, int32_t vp_count,
                 int32_t proc_count, od_move* out, int32_t cap, int32_t* n_out) {
  return guarded([&] {
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    return emit_moves(plan_greedy(l, m, proc_count), out, cap, n_out);
  });
}

int od_refine_swap_lb(const double* loads, int32_t n_loads, const int32_t* map,
                      int32_t vp_count, int32_t proc_count, double tolerance, od_move* out,
                      int32_t cap, int32_t* n_out) {
  return guarded([&] {
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    return emit_moves(plan_refine_swap(l, m, proc_count, tolerance), out, cap, n_out);
  });
}

int od_refine_adjacent_lb(const double* loads, int32_t n_loads, const int32_t* map,
                          int32_t vp_count, int32_t proc_count, double tolerance,
                          int32_t decomposition_kind, int32_t kx, int32_t ky, od_move* out,
                          int32_t cap, int32_t* n_out) {
  return guarded([&] {
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    return emit_moves(plan_refine_adjacent(l, m, proc_count, tolerance, decomposition_kind, kx, ky),
                      out, cap, n_out);
  });
}

static Capacity capacity_of(const int64_t* vp_bytes, int32_t vp_count,
                            const int32_t* bin_of_proc, int32_t proc_count, int32_t n_bins,
                            const int64_t* bin_capacity) {
  if (n_bins < 1) throw ValidationError("capacity: need at least one bin");
  need(vp_bytes, "vp_bytes");
  need(bin_of_proc, "bin_of_proc");
  need(bin_capacity, "bin_capacity");
  Capacity c;
  c.vp_bytes.assign(vp_bytes, vp_bytes + vp_count);
  c.bin_of_proc.assign(bin_of_proc, bin_of_proc + proc_count);
  c.bin_cap.assign(bin_capacity, bin_capacity + n_bins);
  c.validate(vp_count, proc_count);
  return c;
}

int od_greedy_lb_capacity(const double* loads, int32_t n_loads, const int32_t* map,
                          int32_t vp_count, int32_t proc_count, const int64_t* vp_bytes,
                          const int32_t* bin_of_proc, int32_t n_bins,
                          const int64_t* bin_capacity, od_move* out, int32_t cap,
                          int32_t* n_out) {
  return guarded([&] {
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    const Capacity c = capacity_of(vp_bytes, vp_count, bin_of_proc, proc_count, n_bins,
                                   bin_capacity);
    return emit_moves(plan_greedy_capacity(l, m, proc_count, c), out, cap, n_out);
  });
}

int od_refine_swap_lb_capacity(const double* loads, int32_t n_loads, const int32_t* map,
                               int32_t vp_count, int32_t proc_count, double tolerance,
                               const int64_t* vp_bytes, const int32_t* bin_of_proc,
                               int32_t n_bins, const int64_t* bin_capacity, od_move* out,
                               int32_t cap, int32_t* n_out) {
  return guarded([&] {
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    const Capacity c = capacity_of(vp_bytes, vp_count, bin_of_proc, proc_count, n_bins,
                                   bin_capacity);
    return emit_moves(plan_refine_capacity(l, m, proc_count, tolerance, c), out, cap, n_out);
  });
}

static GpuCostModel gpu_of(const od_gpu_model* g) {
  need(g, "gpu model");
  GpuCostModel m;
  m.launch_overhead = g->launch_overhead;
  m.per_item_time = g->per_item_time;
  m.saturation_floor = g->saturation_floor;
  m.h2d_bandwidth = g->h2d_bandwidth;
  m.d2h_bandwidth = g->d2h_bandwidth;
  m.async_overlap_gain = g->async_overlap_gain;
  m.validate();
  return m;
}

int od_kernel_time_sync(const od_kernel_work* work, const od_gpu_model* gpu, double* out) {
  return guarded([&] {
    need(work, "work");
    need(out, "out");
    *out = kernel_time_sync_model(Work{work->work_items, work->serial_depth}, gpu_of(gpu));
  });
}

int od_transfer_time(double bytes, int32_t host_to_device, const od_gpu_model* gpu, double* out) {
  return guarded([&] {
    need(out, "out");
    *out = transfer_time_model(bytes, host_to_device != 0, gpu_of(gpu));
  });
}

int od_node_gpu_schedule(const double* jobs, int32_t n, int32_t mode, const od_gpu_model* gpu,
                         double* out) {
  return guarded([&] {
    need(out, "out");
    if (mode != OD_SYNC && mode != OD_ASYNC) throw ValidationError("unknown launch mode");
    *out = node_gpu_schedule_model(vec_view(jobs, n, "jobs"), mode, gpu_of(gpu));
  });
}

int od_plan_cost(const od_move* moves, int32_t n_moves, const int64_t* data_bytes,
                 int32_t vp_count, int32_t procs_per_node, int32_t nodes,
                 double network_bandwidth, double network_latency, const od_gpu_model* gpu,
                 double* out) {
  return guarded([&] {
    need(out, "out");
    if (n_moves < 0 || vp_count < 0) throw ValidationError("negative count");
    if (n_moves > 0) need(moves, "moves");
    if (vp_count > 0) need(data_bytes, "data_bytes");
    if (network_bandwidth <= 0) throw ValidationError("cluster.network_bandwidth must be > 0");
    if (network_latency < 0) throw ValidationError("cluster.network_latency must be >= 0");
    std::vector<MoveRec> mv(n_moves);
    for (int32_t i = 0; i < n_moves; ++i) mv[i] = {moves[i].vp, moves[i].from, moves[i].to};
    std::vector<int64_t> db(data_bytes, data_bytes + vp_count);
    *out = plan_cost_model(mv, db, procs_per_node, nodes, network_bandwidth, network_latency,
                           gpu_of(gpu));
  });
}

static std::vector<CalibSample> samples_of(const od_kernel_work* work, const double* seconds,
                                           int32_t n) {
  if (n < 0) throw ValidationError("negative count");
  if (n > 0) {
    need(work, "work");
    need(seconds, "seconds");
  }
  std::vector<CalibSample> ss(n);
  for (int32_t i = 0; i < n; ++i) ss[i] = {Work{work[i].work_items, work[i].serial_depth}, seconds[i]};
  return ss;
}

int od_calibrate_gpu(const od_kernel_work* work, const double* seconds, int32_t n,
                     const od_gpu_model* defaults, od_gpu_model* out, double* max_rel_residual) {
  return guarded([&] {
    need(out, "out");
    const GpuFit f = calibrate_gpu_model(samples_of(work, seconds, n), gpu_of(defaults));
    *out = od_gpu_model{f.model.launch_overhead, f.model.per_item_time, f.model.saturation_floor,
                        f.model.h2d_bandwidth, f.model.d2h_bandwidth, f.model.async_overlap_gain};
    if (max_rel_residual) *max_rel_residual = f.max_rel_residual;
  });
}

int od_calibrate_cpu(const od_kernel_work* work, const double* seconds, int32_t n,
                     double* per_item_time) {
  return guarded([&] {
    need(per_item_time, "per_item_time");
    *per_item_time = calibrate_cpu_model(samples_of(work, seconds, n));
  });
}

int od_cpu_time(const od_kernel_work* work, double per_item_time, double* out) {
  return guarded([&] {
    need(work, "work");
    need(out, "out");
    if (per_item_time <= 0) throw ValidationError("cpu model per_item_time must be > 0");
    *out = cpu_time_model(Work{work->work_items, work->serial_depth}, per_item_time);
  });
}

int od_scaling_probe(int32_t n, const int32_t* m_list, int32_t n_m, double inner,
                     const od_gpu_model* gpu, double cpu_per_item, double* cpu_seconds,
                     double* gpu_seconds) {
  return guarded([&] {
    if (n_m < 0) throw ValidationError("negative count");
    if (n_m > 0) {
      need(m_list, "m_list");
      need(cpu_seconds, "cpu_seconds");
      need(gpu_seconds, "gpu_seconds");
    }
    if (cpu_per_item <= 0) throw ValidationError("cpu model per_item_time must be > 0");
    std::vector<double> c, g;
    scaling_probe_model(n, std::vector<int32_t>(m_list, m_list + n_m), inner, gpu_of(gpu),
                        cpu_per_item, c, g);
    std::copy(c.begin(), c.end(), cpu_seconds);
    std::copy(g.begin(), g.end(), gpu_seconds);
  });
}

int od_plan_cost_nvlink(const od_move* moves, int32_t n_moves, const int64_t* data_bytes,
                        int32_t vp_count, int32_t procs_per_gpu, int32_t gpus,
                        double link_bandwidth, double latency, double* out) {
  return guarded([&] {
    need(out, "out");
    if (n_moves < 0 || vp_count < 0) throw ValidationError("negative count");
    if (n_moves > 0) need(moves, "moves");
    if (vp_count > 0) need(data_bytes, "data_bytes");
    std::vector<MoveRec> mv(n_moves);
    for (int32_t i = 0; i < n_moves; ++i) mv[i] = {moves[i].vp, moves[i].from, moves[i].to};
    *out = plan_cost_nvlink_model(mv, std::vector<int64_t>(data_bytes, data_bytes + vp_count),
                                  procs_per_gpu, gpus, link_bandwidth, latency);
  });
}

int od_epoch_decision(const double* loads, int32_t n_loads, const int32_t* map,
                      int32_t vp_count, int32_t proc_count, int32_t epoch_index, int32_t epochs,
                      int32_t* balance_calls, int32_t first_strategy, int32_t later_strategy,
                      double trigger_threshold, double refine_tolerance, int32_t* strategy,
                      od_move* moves, int32_t cap, int32_t* n_moves, double* totals,
                      double* imbalance_before, double* imbalance_after) {
  return guarded([&] {
    need(balance_calls, "balance_calls");
    need(strategy, "strategy");
    if (first_strategy < 0 || first_strategy > 1 || later_strategy < 0 || later_strategy > 1)
      throw ValidationError("unknown strategy");
    if (trigger_threshold < 1.0) throw ValidationError("policy.trigger_threshold must be >= 1");
    if (refine_tolerance < 0.0) throw ValidationError("policy.refine_tolerance must be >= 0");
    auto l = vec_view(loads, n_loads, "loads");
    auto m = map_view(map, vp_count, proc_count);
    Decision d = decide_epoch(l, m, proc_count, epoch_index, epochs, *balance_calls,
                              first_strategy, later_strategy, trigger_threshold,
                              refine_tolerance);
    *strategy = d.strategy;
    if (totals) std::memcpy(totals, d.totals.data(), d.totals.size() * sizeof(double));
    if (imbalance_before) *imbalance_before = d.imbalance_before;
    if (imbalance_after) *imbalance_after = d.imbalance_after;
    return emit_moves(d.plan, moves, cap, n_moves);
  });
}

int od_chunk_neighbor(int32_t kind, int32_t kx, int32_t ky, int32_t vp, int32_t side,
                      int32_t* out) {
  return guarded([&] {
    need(out, "out");
    if (side < 0 || side > 3) throw ValidationError("side must be 0..3");
    if (kx < 1 || ky < 1 || vp < 0 || vp >= (kind == OD_ONE_D ? 1 : kx) * ky)
      throw ValidationError("vp outside the decomposition");
    *out = chunk_neighbor(kind, kx, ky, vp, side);
  });
}

int od_exchange_schedule(const od_subdomain* subs, int32_t vp_count, int32_t kind, int32_t kx,
                         int32_t ky, const int32_t* rank_of_vp, int32_t world, int32_t rank,
                         int64_t per_cell, od_face_xfer* sends, int32_t send_cap,
                         int32_t* n_sends, od_face_xfer* recvs, int32_t recv_cap,
                         int32_t* n_recvs) {
  return guarded([&] {
    if (vp_count < 1) throw ValidationError("vp count must be >= 1");
    if (world < 1 || rank < 0 || rank >= world) throw ValidationError("rank out of range");
    need(subs, "subs");
    need(rank_of_vp, "rank_of_vp");
    need(n_sends, "n_sends");
    need(n_recvs, "n_recvs");
    if ((kind == OD_ONE_D ? ky : kx * ky) != vp_count)
      throw ValidationError("decomposition does not match vp count");
    std::vector<Sub> sv(vp_count);
    std::vector<int32_t> rv(rank_of_vp, rank_of_vp + vp_count);
    for (int32_t v = 0; v < vp_count; ++v) {
      sv[v] = to_sub(subs[v]);
      if (rv[v] < 0 || rv[v] >= world) throw ValidationError("rank id out of range");
    }
    std::vector<FaceXfer> s, r;
    exchange_schedule(sv, kind, kx, ky, rv, world, rank, per_cell, s, r);
    *n_sends = int32_t(s.size());
    *n_recvs = int32_t(r.size());
    if (int32_t(s.size()) > send_cap || int32_t(r.size()) > recv_cap)
      throw ValidationError("face buffer too small");
    auto put = [](const FaceXfer& f) {
      return od_face_xfer{f.peer, f.vp, f.side, f.nbr, f.len, f.lenp, f.offset};
    };
    for (size_t i = 0; i < s.size(); ++i) sends[i] = put(s[i]);
    for (size_t i = 0; i < r.size(); ++i) recvs[i] = put(r[i]);
  });
}

struct od_loaddb {
  SampleStore store;
};

int od_loaddb_create(int32_t vp_count, int32_t async_steps, int32_t sync_steps,
                     od_loaddb** out) {
  return guarded([&] {
    need(out, "out");
    *out = new od_loaddb{SampleStore(vp_count, async_steps, sync_steps)};
  });
}

int od_loaddb_record(od_loaddb* db, const od_sample* s) {
  return guarded([&] {
    need(db, "db");
    need(s, "sample");
    db->store.add(s->vp, s->step, s->mode, s->value);
  });
}

int od_loaddb_clear(od_loaddb* db) {
  return guarded([&] {
    need(db, "db");
    db->store.reset();
  });
}

int od_loaddb_size(const od_loaddb* db, int32_t* n) {
  return guarded([&] {
    need(db, "db");
    need(n, "n");
    *n = int32_t(db->store.size());
  });
}

int od_loaddb_epoch_loads(const od_loaddb* db, double* out) {
  return guarded([&] {
    need(db, "db");
    auto m = db->store.sync_means();
    if (!m.empty()) need(out, "out");
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  });
}

void od_loaddb_destroy(od_loaddb* db) { delete db; }

}  // extern "C"
