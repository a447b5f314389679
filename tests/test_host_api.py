"""Host-side API (no GPU): the reference's validation and known answers for
GridSpec, TimestepController, choose_dt, SimulationConfig, make_kernel and the
descriptor table (reference tests test_grid.py, test_driver.py:19-60,
test_kernels.py:21-33, 301-322)."""

from fractions import Fraction

import numpy as np
import pytest

from paper_1308_1464_b200 import (DEFAULT_IC, DESCRIPTORS, KERNEL_NAMES, AcousticsParams,
                                  BoundaryCondition, Cuda, EulerParams, GridSpec,
                                  ShallowWaterParams, SimulationConfig, StateField,
                                  TimestepController, allocate_fields, choose_dt,
                                  initial_condition, make_kernel)


def gas_spec(nx, ny):
    return GridSpec(nx=nx, ny=ny, dx=1.0 / nx, dy=1.0 / ny, num_eqn=4)


class TestGrid:
    def test_allocation_shapes(self):
        spec = GridSpec(nx=4, ny=3, dx=0.1, dy=0.1, num_ghost=2, num_eqn=3)
        state, aux = allocate_fields(spec)
        assert state.data.shape == (3, 8, 7)
        assert aux.data.shape == (0, 8, 7)
        assert state.data.strides[0] == state.data.itemsize   # component fastest (F order)

    @pytest.mark.parametrize("bad", [
        dict(nx=0, ny=3, dx=0.1, dy=0.1), dict(nx=3, ny=-1, dx=0.1, dy=0.1),
        dict(nx=3, ny=3, dx=0.0, dy=0.1), dict(nx=3, ny=3, dx=0.1, dy=-0.5),
        dict(nx=3, ny=3, dx=0.1, dy=0.1, num_ghost=0),
        dict(nx=3, ny=3, dx=0.1, dy=0.1, num_eqn=0),
        dict(nx=3, ny=3, dx=0.1, dy=0.1, num_aux=-1)])
    def test_invalid_spec_rejected(self, bad):
        with pytest.raises(ValueError):
            GridSpec(**bad)

    def test_checked_accessor(self):
        spec = GridSpec(nx=4, ny=3, dx=1.0, dy=1.0, num_ghost=1, num_eqn=2)
        state = StateField(spec)
        state.value(1, -1, 3)
        for comp, i, j in [(2, 0, 0), (0, -2, 0), (0, 5, 0), (0, 0, -2), (0, 0, 4)]:
            with pytest.raises(IndexError):
                state.value(comp, i, j)

    def test_copy_is_independent(self):
        spec = GridSpec(nx=3, ny=3, dx=1.0, dy=1.0, num_eqn=1)
        s = StateField(spec)
        s.interior[:] = 1.0
        d = s.copy()
        d.interior[:] = 2.0
        assert np.all(s.interior == 1.0)


class TestChooseDt:
    # reference test_driver.py:19-45
    def test_symmetric_speeds(self):
        assert choose_dt(1.0, 1.0, 0.01, 0.01, TimestepController(0.9)) == \
            pytest.approx(0.0045, rel=1e-12)

    def test_pure_x_motion(self):
        assert choose_dt(2.0, 0.0, 0.1, 0.1, TimestepController(0.5)) == \
            pytest.approx(0.025, rel=1e-12)

    def test_fixed_dt_bypasses_formula(self):
        assert choose_dt(0.0, 0.0, 0.1, 0.1, TimestepController(fixed_dt=1e-3)) == 1e-3

    def test_stationary_is_an_error(self):
        with pytest.raises(ValueError, match="stationary"):
            choose_dt(0.0, 0.0, 0.1, 0.1, TimestepController())

    def test_clamps(self):
        ctl = TimestepController(cfl_target=0.9, dt_max=1e-3)
        assert choose_dt(1.0, 0.0, 1.0, 1.0, ctl) == 1e-3
        assert choose_dt(1.0, 0.0, 1.0, 1.0, ctl, remaining=1e-4) == 1e-4

    @pytest.mark.parametrize("cfl", [0.0, 1.0, -0.1, 1.5])
    def test_cfl_range(self, cfl):
        with pytest.raises(ValueError):
            TimestepController(cfl_target=cfl)

    def test_native_ctl_uses_nan_for_none(self):
        c = TimestepController(0.8, dt_max=0.5).native(remaining=0.25)
        assert c.cfl == 0.8 and c.dt_max == 0.5 and c.remaining == 0.25
        assert np.isnan(c.fixed_dt) and np.isnan(c.t_final)


class TestConfig:
    def test_exactly_one_stop_rule(self):
        with pytest.raises(ValueError, match="exactly one"):
            SimulationConfig(spec=gas_spec(8, 8), kernel="euler", ic="euler-sod-x")
        with pytest.raises(ValueError, match="exactly one"):
            SimulationConfig(spec=gas_spec(8, 8), kernel="euler", ic="euler-sod-x",
                             t_final=1.0, num_steps=5)

    def test_unknown_kernel_and_limiter(self):
        with pytest.raises(ValueError, match="unknown kernel"):
            SimulationConfig(spec=gas_spec(8, 8), kernel="maxwell", ic="x", num_steps=1)
        with pytest.raises(ValueError, match="unknown limiter"):
            SimulationConfig(spec=gas_spec(8, 8), kernel="euler", ic="euler-sod-x",
                             num_steps=1, order=2, limiter="vanleer")

    def test_no_cpu_backend(self):
        with pytest.raises(TypeError):
            SimulationConfig(spec=gas_spec(8, 8), kernel="euler", ic="euler-sod-x",
                             num_steps=1, backend="serial")

    def test_cuda_backend_precision(self):
        with pytest.raises(ValueError):
            Cuda(precision="f16")


class TestKernels:
    def test_descriptor_table(self):
        assert DESCRIPTORS["acoustics-const"].num_eqn == 3
        assert DESCRIPTORS["acoustics-const"].num_waves == 2
        assert DESCRIPTORS["acoustics-var"].num_aux == 2
        assert DESCRIPTORS["euler"].num_waves == 3
        assert DESCRIPTORS["euler-hlle"].num_waves == 2
        assert DESCRIPTORS["shallow-water-roe"].num_eqn == 3
        assert DESCRIPTORS["euler"].arithmetic_intensity == Fraction(1)
        assert set(DEFAULT_IC) == set(KERNEL_NAMES)

    def test_make_kernel_binding(self):
        assert make_kernel("euler").params["gamma"] == 1.4
        assert make_kernel("shallow-water-roe").params["grav"] == 9.81
        k = make_kernel("acoustics-const", rho=2.0, bulk=8.0)
        assert k.native_params()[:2] == [2.0, 8.0]
        with pytest.raises(ValueError, match="unknown kernel"):
            make_kernel("burgers")
        with pytest.raises(ValueError, match="unexpected"):
            make_kernel("euler", gamma=1.4, mach=3)

    def test_param_validation(self):
        with pytest.raises(ValueError):
            AcousticsParams(0.0, 1.0)
        with pytest.raises(ValueError):
            EulerParams(1.0)
        with pytest.raises(ValueError):
            ShallowWaterParams(0.0)
        assert AcousticsParams(2.0, 8.0).sound_speed == 2.0

    def test_initial_conditions(self):
        spec = gas_spec(8, 4)
        state, _, params = initial_condition("euler-sod-x", spec)
        assert params == {"gamma": 1.4}
        assert tuple(state.interior[:, 0, 0]) == (1.0, 0.0, 0.0, 2.5)
        assert tuple(state.interior[:, -1, 0]) == (0.125, 0.0, 0.0, 0.25)
        with pytest.raises(ValueError, match="unknown initial condition"):
            initial_condition("vortex", spec)
        with pytest.raises(ValueError, match="num_eqn"):
            initial_condition("acoustics-pulse", spec)
        spec = GridSpec(nx=8, ny=4, dx=1 / 8, dy=1 / 4, num_eqn=3, num_aux=2)
        _, aux, _ = initial_condition("acoustics-var-interface", spec)
        assert np.all(aux.interior[1, :4] == 1.0) and np.all(aux.interior[1, 4:] == 3.0)

    def test_boundary_enum(self):
        assert BoundaryCondition("periodic") is BoundaryCondition.PERIODIC
