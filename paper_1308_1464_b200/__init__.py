"""B200-native 2D wave-propagation step — drop-in for the hot path of the
reference ``wavesweep`` package (arXiv 1308.1464, ManyClaw).

Public surface mirrors reference ``wavesweep/__init__.py``: grid, kernels,
sweep errors, and the driver's step/run.  Everything that computes runs in
CUDA (``paper_1308_1464_b200/csrc``) behind the C ABI in
``include/wavestep.h``; there is no CPU backend.
"""

from .device import Cuda, DeviceGrid
from .driver import (DEFAULT_IC, SimulationConfig, StepReport, TimestepController,
                     choose_dt, initial_condition, run, step)
from .grid import (AuxField, BoundaryCondition, GridSpec, StateField, allocate_fields,
                   fill_ghost)
from .kernels import (DESCRIPTORS, KERNEL_NAMES, AcousticsParams, Direction, EulerParams,
                      Kernel, KernelDescriptor, KernelError, RiemannResult,
                      ShallowWaterParams, make_kernel)
from .sweep import CellWise, RowWise, SweepError, Tiled

__version__ = "0.1.0"
