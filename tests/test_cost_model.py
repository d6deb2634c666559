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
