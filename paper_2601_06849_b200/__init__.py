"""paper_2601_06849_b200 — B200-native ETD2RK-DS spectral time stepping (arXiv 2601.06849).

The hot path (the reference's etd2rkds_step_2d/3d and etd2rkds_step_system,
/root/reference/proj/core/src/stepper.cpp:182-257, system_stepper.cpp:74-114)
runs in hand-written sm_100a CUDA (``csrc/``) behind the C-ABI
``include/etd_b200.h``; this Python layer mirrors the reference stepper API.
"""
from .etd import (BackendKind, ConfigError, DeviceError, DeviceSource, Grid, MemoryGuardError, NumericsError,
                  PadeFamily, SourceKind, StepperAbort, StepperPlan, StepperState, SystemPlan, SystemState,
                  advance, etd2rkds_step_2d, etd2rkds_step_3d, etd2rkds_reference_step, etd2rk_nonsplit_step, phi1, phi2,
                  allen_cahn_cubic, allen_cahn_manufactured, singular, build_grid, etd2rkds_step_system, fhn_classic, fhn_cubic,
                  fill_config_ic, lib, make_plan, make_system_plan, poly3, setup_axis, setup_dvector,
                  setup_scheme, unit_box_grid, zslab_partition, nccl_unique_id, group_step, plan_device_bytes)
from . import configs, harness

__all__ = [n for n in dir() if not n.startswith("_")]
