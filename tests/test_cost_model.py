"""The reference's analytic cost functions (gpu_cost.hpp:50-80,
balancer.hpp:157-175), kept with identical arithmetic next to the measured B200
path: unit-test vectors of test_gpucost.cpp / test_balancer.cpp and random
agreement with the reference itself."""
import numpy as np
import pytest

import paper_1310_4218_b200 as od
from oracle import ref as oref


def test_kernel_time_hinge_and_floor():  # test_gpucost.cpp:8-16
    g = od.GpuModel(launch_overhead=1e-3, per_item_time=1e-9, saturation_floor=5e-3)
    assert od.kernel_time_sync(od.KernelWork(0, 0), g) == 0.0
    assert od.kernel_time_sync(od.KernelWork(10, 1), g) == pytest.approx(5e-3)
    assert od.kernel_time_sync(od.KernelWork(1e7, 1), g) == pytest.approx(1e-3 + 1e-2)


def test_directional_bandwidth():  # test_gpucost.cpp:24-33
    g = od.GpuModel(h2d_bandwidth=4e9, d2h_bandwidth=8e9)
    assert od.transfer_time(8e9, od.TransferDirection.HostToDevice, g) == pytest.approx(2.0)
    assert od.transfer_time(8e9, od.TransferDirection.DeviceToHost, g) == pytest.approx(1.0)
    assert od.transfer_time(0, od.TransferDirection.DeviceToHost, g) == 0.0
    with pytest.raises(od.ValidationError):
        od.transfer_time(-1, od.TransferDirection.DeviceToHost, g)


def test_node_schedule():  # test_gpucost.cpp:35-46 and test_properties.cpp:36-49
    g = od.GpuModel(async_overlap_gain=0.1)
    assert od.node_gpu_schedule([1.0, 2.0, 3.0], od.LaunchMode.Sync, g) == pytest.approx(6.0)
    assert od.node_gpu_schedule([1.0, 2.0, 3.0], od.LaunchMode.Async, g) == pytest.approx(5.4)
    assert od.node_gpu_schedule([0.1, 5.0], od.LaunchMode.Async, g) == pytest.approx(5.0)
    rng = np.random.default_rng(7)
    for _ in range(300):
        jobs = rng.uniform(0, 5, int(rng.integers(1, 13)))
        a = od.node_gpu_schedule(jobs, od.LaunchMode.Async, g)
        assert a <= od.node_gpu_schedule(jobs, od.LaunchMode.Sync, g) + 1e-12
        assert a >= jobs.max() - 1e-12


def test_plan_cost_kat():  # test_balancer.cpp:143-161
    g = od.GpuModel(h2d_bandwidth=6e9, d2h_bandwidth=6e9)
    b = [6_000_000_000] * 4
    assert od.plan_cost(od.MigrationPlan([od.Move(0, 0, 1)]), b, 2, 2, g) == pytest.approx(2.0)
    assert od.plan_cost(od.MigrationPlan([od.Move(0, 0, 2)]), b, 2, 2, g) == \
        pytest.approx(1.0 + 6.0 / 5.0 + 1e-5)
    assert od.plan_cost(od.MigrationPlan(), b, 2, 2, g) == 0.0


@pytest.mark.skipif(not oref.available(), reason="oracle/_ref not built")
def test_cost_functions_match_reference_random():
    rng = np.random.default_rng(11)
    for _ in range(200):
        g = od.GpuModel(float(rng.uniform(0, 1e-3)), float(rng.uniform(1e-10, 1e-8)),
                        float(rng.uniform(0, 1e-2)), float(rng.uniform(1e9, 1e10)),
                        float(rng.uniform(1e9, 1e10)), float(rng.uniform(0, 0.5)))
        items, depth = float(rng.uniform(0, 1e7)), float(rng.uniform(0, 100))
        assert od.kernel_time_sync(od.KernelWork(items, depth), g) == \
            oref.kernel_time_sync(items, depth, g)
        nb = float(rng.uniform(0, 1e9))
        assert od.transfer_time(nb, od.TransferDirection.HostToDevice, g) == \
            oref.transfer_time(nb, 1, g)
        jobs = rng.uniform(0, 3, int(rng.integers(1, 9)))
        for mode in (0, 1):
            assert od.node_gpu_schedule(jobs, od.LaunchMode(mode), g) == \
                oref.node_gpu_schedule(jobs, mode, g)
        nodes, ppn = int(rng.integers(1, 4)), int(rng.integers(1, 3))
        P, K = nodes * ppn, int(rng.integers(2, 20))
        m = rng.integers(0, P, K)
        loads = rng.uniform(0.1, 5, K)
        plan = od.greedy_lb(loads, od.Mapping(proc_count=P, assignment=m))
        by = rng.integers(1, 10**9, K)
        assert od.plan_cost(plan, by, ppn, nodes, g, 5e9, 1e-5) == \
            oref.plan_cost([tuple(x) for x in plan.moves], by, nodes, ppn, 5e9, 1e-5, g)


# ------------------------------------------------------------------ calibration
def _rows(samples):
    return [(s.work.work_items, s.work.serial_depth, s.seconds) for s in samples]


def test_gpu_calibration_round_trips_exact_hinge_data():  # test_gpucost.cpp:48-65
    truth = od.GpuModel(launch_overhead=2e-4, per_item_time=5e-12, saturation_floor=0.15)
    samples = [od.CalibrationSample(od.KernelWork(i, 1.0),
                                    od.kernel_time_sync(od.KernelWork(i, 1.0), truth))
               for i in (1e9, 2e10, 6e10, 1e11, 2e11)]
    fit = od.calibrate_gpu(samples)
    assert fit.model.per_item_time == pytest.approx(truth.per_item_time, rel=1e-6)
    assert fit.model.launch_overhead == pytest.approx(truth.launch_overhead, rel=1e-6)
    assert fit.model.saturation_floor == pytest.approx(truth.saturation_floor, rel=1e-6)
    assert fit.max_relative_residual < 1e-9


def test_cpu_calibration_round_trips_linear_data():  # test_gpucost.cpp:67-74
    truth = od.CpuModel(3.3e-9)
    samples = [od.CalibrationSample(od.KernelWork(i, 2.0), od.cpu_time(od.KernelWork(i, 2.0), truth))
               for i in (1e8, 3e8, 9e8)]
    assert od.calibrate_cpu(samples).per_item_time == pytest.approx(3.3e-9, rel=1e-9)


def test_bundled_probe_fit_and_table():  # test_gpucost.cpp:76-82, acceptance.cpp:113-137
    fit = od.calibrate_gpu(od.reference_gpu_probe_samples())
    assert fit.max_relative_residual <= 0.25
    cpu = od.calibrate_cpu(od.reference_cpu_probe_samples())
    for s in od.reference_cpu_probe_samples():
        assert od.cpu_time(s.work, cpu) == pytest.approx(s.seconds, rel=0.10)
    rows = od.scaling_probe(1024, [512, 256, 128, 64, 32], 2e5, fit.model, cpu)
    assert len(rows) == 5
    for a, b in zip(rows, rows[1:]):
        assert b.cpu_seconds < a.cpu_seconds
        assert b.gpu_seconds <= a.gpu_seconds + 1e-12
    for r, t in zip(rows, (54.41, 27.1, 13.45)):
        assert abs(r.cpu_seconds - t) / t <= 0.10
    for r, t in zip(rows, (0.82, 0.49, 0.33, 0.17, 0.18)):
        assert abs(r.gpu_seconds - t) / t <= 0.25
    assert abs(rows[4].gpu_seconds - rows[3].gpu_seconds) / rows[3].gpu_seconds <= 0.10
    with pytest.raises(od.ValidationError):
        od.scaling_probe(1024, [], 2e5, fit.model, cpu)


def test_calibration_input_validation():  # test_gpucost.cpp:84-89
    S, W = od.CalibrationSample, od.KernelWork
    with pytest.raises(od.ValidationError):
        od.calibrate_gpu([S(W(1e9, 1), 0.5)])
    with pytest.raises(od.ValidationError):
        od.calibrate_gpu([S(W(1e9, 1), 0.5), S(W(2e9, 1), 0.0), S(W(3e9, 1), 1.0)])
    with pytest.raises(od.ValidationError):
        od.calibrate_cpu([])
    with pytest.raises(od.ValidationError):  # identical work: no line through the points
        od.calibrate_gpu([S(W(1e9, 1), 0.5), S(W(1e9, 1), 0.9), S(W(1e9, 1), 1.3)])


def test_calibration_bit_exact_with_reference():
    """calibrate_gpu (two-stage fit + Nelder-Mead), calibrate_cpu and
    scaling_probe agree bit for bit with the reference on its bundled probe
    samples and on random noisy/saturated/exact sample sets."""
    d = od.GpuModel()
    for samples in (od.reference_gpu_probe_samples(), od.reference_cpu_probe_samples()):
        fit = od.calibrate_gpu(samples, d)
        m, res = oref.calibrate_gpu(_rows(samples), d)
        got = [fit.model.launch_overhead, fit.model.per_item_time, fit.model.saturation_floor,
               fit.model.h2d_bandwidth, fit.model.d2h_bandwidth, fit.model.async_overlap_gain]
        assert got == m and fit.max_relative_residual == res
        assert od.calibrate_cpu(samples).per_item_time == oref.calibrate_cpu(_rows(samples))
    rng = np.random.default_rng(1310)
    for case in range(150):
        n = int(rng.integers(3, 9))
        items = rng.uniform(1e8, 1e11, n) * (rng.integers(1, 3, n) if case % 5 == 0 else 1)
        depth = rng.choice([1.0, 2.0, 64.0, 2e5], n)
        g = od.GpuModel(launch_overhead=rng.uniform(0, 1e-3), per_item_time=rng.uniform(1e-13, 1e-11),
                        saturation_floor=rng.uniform(0, 0.5) if case % 3 else 0.0)
        t = np.array([od.kernel_time_sync(od.KernelWork(a, b), g) for a, b in zip(items, depth)])
        if case % 4:
            t = t * rng.uniform(0.8, 1.25, n)  # measurement noise
        samples = [od.CalibrationSample(od.KernelWork(a, b), float(s))
                   for a, b, s in zip(items, depth, t)]
        try:
            mine = od.calibrate_gpu(samples, d)
        except od.ValidationError:
            with pytest.raises(oref.RefError):
                oref.calibrate_gpu(_rows(samples), d)
            continue
        m, res = oref.calibrate_gpu(_rows(samples), d)
        assert [mine.model.launch_overhead, mine.model.per_item_time,
                mine.model.saturation_floor] == m[:3], case
        assert mine.max_relative_residual == res
        assert od.calibrate_cpu(samples).per_item_time == oref.calibrate_cpu(_rows(samples))
        ms = [int(x) for x in rng.integers(3, 600, int(rng.integers(1, 7)))]
        rows = od.scaling_probe(1024, ms, 2e5, mine.model, od.CpuModel(3e-9))
        c, gg = oref.scaling_probe(1024, ms, 2e5, mine.model, 3e-9)
        assert [r.cpu_seconds for r in rows] == c and [r.gpu_seconds for r in rows] == gg


def test_plan_cost_nvlink():
    M, P = od.Move, od.MigrationPlan
    b = [100e9 // 100] * 8  # 1 GB per chunk
    bw, lat = 500e9, 1e-5
    assert od.plan_cost_nvlink(P([]), b, 1, 4, bw, lat) == 0.0
    # a move between processors of one GPU is free
    assert od.plan_cost_nvlink(P([M(0, 0, 1)]), b, 2, 2, bw, lat) == 0.0
    one = od.plan_cost_nvlink(P([M(0, 0, 1)]), b, 1, 2, bw, lat)
    assert one == pytest.approx(1e9 / bw + lat)
    # disjoint pairs copy concurrently; two moves out of one GPU serialise on its port
    par = od.plan_cost_nvlink(P([M(0, 0, 1), M(1, 2, 3)]), b, 1, 4, bw, lat)
    ser = od.plan_cost_nvlink(P([M(0, 0, 1), M(1, 0, 2)]), b, 1, 4, bw, lat)
    assert par == pytest.approx(one) and ser == pytest.approx(2e9 / bw + 2 * lat)
    # a swap: each GPU sends one and receives one chunk
    assert od.plan_cost_nvlink(P([M(0, 0, 1), M(1, 1, 0)]), b, 1, 2, bw, lat) == \
        pytest.approx(1e9 / bw + 2 * lat)
    with pytest.raises(od.ValidationError):
        od.plan_cost_nvlink(P([M(0, 0, 9)]), b, 1, 4, bw, lat)
    with pytest.raises(od.ValidationError):
        od.plan_cost_nvlink(P([]), b, 1, 4, 0.0, lat)
