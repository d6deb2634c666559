// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.  A thin extern "C" wrapper that
// compiles the REFERENCE simulator's own headers, where they lie under
// /root/reference/proj/include/overdeck/, into oracle/_ref/libodref.so
// (recipe: oracle/Makefile).  No reference source is copied into this repo;
// this file only calls the reference's public API so the tests can compare
// the B200 library against the reference implementation itself:
//   greedy_lb / refine_swap_lb           balancer.hpp:36-152
//   decompose_1d / decompose_2d          workload.hpp:100-139
//   init_load_field / advect_load_field  workload.hpp:160-195
//   physics_work / jacobi_work           workload.hpp:199-210
//   initial_block_mapping / apply_plan   cluster.hpp:115-139
//   proc_loads / imbalance_ratio         cluster.hpp:142-157
//   LoadDB / epoch_loads                 measurement.hpp:40-91
//   run_experiment + render_report       engine.hpp:357, report.hpp:69
//   kernel_time_sync / transfer_time / node_gpu_schedule / plan_cost
//                                        gpu_cost.hpp:50-80, balancer.hpp:157-175
//   calibrate_gpu / calibrate_cpu / cpu_time / scaling_probe
//                                        gpu_cost.hpp:56-58,187-261, engine.hpp:363-373
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "overdeck/config.hpp"
#include "overdeck/presets.hpp"
#include "overdeck/report.hpp"

using namespace overdeck;

namespace {
thread_local std::string g_err;

template <typename F>
int wrap(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const RuntimeFault& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

Mapping make_mapping(const int* map, int K, int P) {
  Mapping m(K, P);
  for (int v = 0; v < K; ++v) m.assign(v, map[v]);
  return m;
}

void put_plan(const MigrationPlan& p, int* out, int cap, int* n) {
  *n = static_cast<int>(p.moves.size());
  if (*n > cap) throw ValidationError("plan buffer too small");
  for (int i = 0; i < *n; ++i) {
    out[3 * i] = p.moves[i].vp;
    out[3 * i + 1] = p.moves[i].from;
    out[3 * i + 2] = p.moves[i].to;
  }
}

int put_string(const std::string& s, char* out, long cap) {
  if (static_cast<long>(s.size()) + 1 > cap) {
    g_err = "output buffer too small: need " + std::to_string(s.size() + 1);
    return 5;
  }
  std::memcpy(out, s.data(), s.size() + 1);
  return 0;
}

void put_subs(const std::vector<SubDomain>& subs, long long* out) {
  for (size_t i = 0; i < subs.size(); ++i) {
    out[6 * i] = subs[i].owner_vp;
    out[6 * i + 1] = subs[i].x_begin;
    out[6 * i + 2] = subs[i].x_end;
    out[6 * i + 3] = subs[i].y_begin;
    out[6 * i + 4] = subs[i].y_end;
    out[6 * i + 5] = subs[i].boundary_cells;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_greedy_lb(const double* loads, int n_loads, const int* map, int K, int P, int* out,
                  int cap, int* n) {
  return wrap([&] {
    put_plan(greedy_lb(LoadVector(loads, loads + n_loads), make_mapping(map, K, P)), out, cap, n);
  });
}

int ref_refine_swap_lb(const double* loads, int n_loads, const int* map, int K, int P,
                       double tol, int* out, int cap, int* n) {
  return wrap([&] {
    put_plan(refine_swap_lb(LoadVector(loads, loads + n_loads), make_mapping(map, K, P), tol),
             out, cap, n);
  });
}

int ref_decompose_1d(int nx, int ny, int k, long long* out) {
  return wrap([&] { put_subs(decompose_1d(Domain{nx, ny, 1, 1}, k), out); });
}

int ref_decompose_2d(int nx, int ny, int kx, int ky, long long* out) {
  return wrap([&] { put_subs(decompose_2d(Domain{nx, ny, 1, 1}, kx, ky), out); });
}

int ref_initial_block_mapping(int K, int P, int* out) {
  return wrap([&] {
    Mapping m = initial_block_mapping(K, P);
    for (int v = 0; v < K; ++v) out[v] = m.proc_of(v);
  });
}

int ref_apply_plan(const int* map, int K, int P, const int* moves, int n, int* out) {
  return wrap([&] {
    MigrationPlan plan;
    for (int i = 0; i < n; ++i) plan.moves.push_back({moves[3 * i], moves[3 * i + 1], moves[3 * i + 2]});
    Mapping r = apply_plan(make_mapping(map, K, P), plan);
    for (int v = 0; v < K; ++v) out[v] = r.proc_of(v);
  });
}

int ref_proc_loads(const double* loads, int n_loads, const int* map, int K, int P, double* out) {
  return wrap([&] {
    auto t = proc_loads(LoadVector(loads, loads + n_loads), make_mapping(map, K, P));
    std::copy(t.begin(), t.end(), out);
  });
}

int ref_imbalance_ratio(const double* totals, int n, double* out) {
  return wrap([&] { *out = imbalance_ratio(std::vector<double>(totals, totals + n)); });
}

// pattern 0 uniform, 1 static_node0 (node0 tiles given as 4-tuples), 2 upper half
int ref_init_load_field(int nx, int ny, int pattern, double heavy, double light,
                        const int* node0, int n_node0, double* out) {
  return wrap([&] {
    std::vector<SubDomain> subs;
    for (int i = 0; i < n_node0; ++i)
      subs.push_back({0, node0[4 * i], node0[4 * i + 1], node0[4 * i + 2], node0[4 * i + 3], 0});
    LoadPattern p = pattern == 0 ? LoadPattern::Uniform
                    : pattern == 1 ? LoadPattern::StaticNode0
                                   : LoadPattern::UpperHalfHeavy;
    LoadField f = init_load_field(Domain{nx, ny, 1, 1}, p, heavy, light, subs);
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) out[static_cast<size_t>(y) * nx + x] = f.at(x, y);
  });
}

static LoadField field_from(const double* c, int nx, int ny) {
  LoadField f(nx, ny);
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) f.set(x, y, c[static_cast<size_t>(y) * nx + x]);
  return f;
}

int ref_advect_load_field(const double* c, int nx, int ny, int shift, double* out) {
  return wrap([&] {
    LoadField r = advect_load_field(field_from(c, nx, ny), shift);
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) out[static_cast<size_t>(y) * nx + x] = r.at(x, y);
  });
}

// physics_work(sub).{work_items, serial_depth} for a rectangle of field c
int ref_physics_work(const double* c, int nx, int ny, int x0, int x1, int y0, int y1, int mzp,
                     double* items, double* depth) {
  return wrap([&] {
    SubDomain s{0, x0, x1, y0, y1, 0};
    KernelWork w = physics_work(s, field_from(c, nx, ny), mzp);
    *items = w.work_items;
    *depth = w.serial_depth;
  });
}

int ref_jacobi_work(int x0, int x1, int y0, int y1, int nz, int fields, double* items,
                    double* depth) {
  return wrap([&] {
    KernelWork w = jacobi_work(SubDomain{0, x0, x1, y0, y1, 0}, nz, fields);
    *items = w.work_items;
    *depth = w.serial_depth;
  });
}

// samples: n rows of (vp, step, mode) ints + values; returns the epoch loads
int ref_epoch_loads(int K, int async_steps, int sync_steps, const int* rows, const double* vals,
                    int n, double* out) {
  return wrap([&] {
    LoadDB db(K, MeasurementWindow{async_steps, sync_steps});
    for (int i = 0; i < n; ++i)
      db.record({rows[3 * i], rows[3 * i + 1],
                 rows[3 * i + 2] == 0 ? LaunchMode::Sync : LaunchMode::Async, vals[i]});
    auto l = epoch_loads(db);
    std::copy(l.begin(), l.end(), out);
  });
}

static GpuModel gm(const double* g) {
  GpuModel m;
  m.launch_overhead = g[0];
  m.per_item_time = g[1];
  m.saturation_floor = g[2];
  m.h2d_bandwidth = g[3];
  m.d2h_bandwidth = g[4];
  m.async_overlap_gain = g[5];
  return m;
}

int ref_kernel_time_sync(double items, double depth, const double* g, double* out) {
  return wrap([&] { *out = kernel_time_sync(KernelWork{items, depth}, gm(g)); });
}

int ref_transfer_time(double bytes, int h2d, const double* g, double* out) {
  return wrap([&] {
    *out = transfer_time(bytes, h2d ? TransferDirection::HostToDevice
                                    : TransferDirection::DeviceToHost, gm(g));
  });
}

int ref_node_gpu_schedule(const double* jobs, int n, int mode, const double* g, double* out) {
  return wrap([&] {
    *out = node_gpu_schedule(std::vector<double>(jobs, jobs + n),
                             mode == 0 ? LaunchMode::Sync : LaunchMode::Async, gm(g));
  });
}

int ref_plan_cost(const int* moves, int n, const long long* bytes, int K, int nodes, int ppn,
                  double bw, double lat, const double* g, double* out) {
  return wrap([&] {
    MigrationPlan plan;
    for (int i = 0; i < n; ++i) plan.moves.push_back({moves[3 * i], moves[3 * i + 1], moves[3 * i + 2]});
    std::vector<VirtualProcess> vps(K);
    for (int v = 0; v < K; ++v) vps[v].data_bytes = bytes[v];
    ClusterState cl = build_cluster(ClusterSpec{nodes, ppn, 1, bw, lat});
    *out = plan_cost(plan, vps, cl, gm(g));
  });
}

static std::vector<CalibrationSample> calib(const double* items, const double* depth,
                                            const double* sec, int n) {
  std::vector<CalibrationSample> v;
  for (int i = 0; i < n; ++i) v.push_back({KernelWork{items[i], depth[i]}, sec[i]});
  return v;
}

int ref_calibrate_gpu(const double* items, const double* depth, const double* sec, int n,
                      const double* defaults, double* out, double* residual) {
  return wrap([&] {
    GpuCalibration c = calibrate_gpu(calib(items, depth, sec, n), gm(defaults));
    out[0] = c.model.launch_overhead;
    out[1] = c.model.per_item_time;
    out[2] = c.model.saturation_floor;
    out[3] = c.model.h2d_bandwidth;
    out[4] = c.model.d2h_bandwidth;
    out[5] = c.model.async_overlap_gain;
    *residual = c.max_relative_residual;
  });
}

int ref_calibrate_cpu(const double* items, const double* depth, const double* sec, int n,
                      double* out) {
  return wrap([&] { *out = calibrate_cpu(calib(items, depth, sec, n)).per_item_time; });
}

int ref_scaling_probe(int n, const int* m, int nm, double inner, const double* g, double cpu,
                      double* cpu_out, double* gpu_out) {
  return wrap([&] {
    auto rows = scaling_probe(n, std::vector<int>(m, m + nm), inner, gm(g), CpuModel{cpu});
    for (size_t i = 0; i < rows.size(); ++i) {
      cpu_out[i] = rows[i].cpu_seconds;
      gpu_out[i] = rows[i].gpu_seconds;
    }
  });
}

// Runs the reference simulator on a JSON config (config.hpp:101) and returns
// render_report's JSON plus the per-epoch mapping and the initial subdomains.
int ref_run_json(const char* config_json, char* out, long cap) {
  std::string doc;
  const int rc = wrap([&] {
    const ExperimentConfig cfg = config_from_json(nlohmann::json::parse(config_json));
    Engine eng(cfg);
    nlohmann::json subs = nlohmann::json::array();
    for (const auto& s : eng.subdomains())
      subs.push_back({s.owner_vp, s.x_begin, s.x_end, s.y_begin, s.y_end, s.boundary_cells});
    const Timeline tl = eng.run();
    nlohmann::json rep = nlohmann::json::parse(render_report(tl, ReportFormat::Json));
    nlohmann::json maps = nlohmann::json::array();
    nlohmann::json strategies = nlohmann::json::array();
    nlohmann::json moves = nlohmann::json::array();
    for (const auto& e : tl.epochs) {
      std::vector<int> m;
      for (int v = 0; v < e.mapping.vp_count(); ++v) m.push_back(e.mapping.proc_of(v));
      maps.push_back(m);
      nlohmann::json mv = nlohmann::json::array();
      for (const auto& x : e.plan.moves) mv.push_back({x.vp, x.from, x.to});
      moves.push_back(mv);
    }
    rep["mappings"] = maps;
    rep["moves"] = moves;
    rep["subdomains"] = subs;
    rep["csv"] = render_report(tl, ReportFormat::Csv);
    doc = rep.dump();
  });
  if (rc) return rc;
  return put_string(doc, out, cap);
}

int ref_preset_json(const char* name, char* out, long cap) {
  std::string doc;
  const int rc = wrap([&] { doc = config_to_json(preset(name)).dump(); });
  if (rc) return rc;
  return put_string(doc, out, cap);
}

}  // extern "C"
