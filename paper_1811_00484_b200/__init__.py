"""B200-native Tucker-compressed VIE matvec (arXiv 1811.00484 hot path).

The compute lives in libvie_b200.so (hand-written sm_100a CUDA behind the C ABI
in include/vie_b200.h); ``vie`` mirrors the reference operator API over it.
"""
from .vie import (KIND_K, KIND_N, PWC, PWL, DftService, EmbeddedSpectrum, GmresConfig, GmresResult, TuckerForm,
                  VieError, apply_operator, apply_operator_batch, apply_system, build_operator_spectra, component_table, gmres, lib,
                  ncur, tucker_compress, RULE_ENERGY, RULE_SIGMA_MAX, DielectricMap, Fields, PlaneWave,
                  PostProcess, VoxelGrid, build_rhs, postprocess, recover_fields,
                  SolveReport, solve_scene, tucker_cp_form, gmres_map, ApplyTimings, apply_operator_timed,
                  KIND_G, QuadratureSpec, assemble_defining_tensor, assemble_operator, self_static_term,
                  set_strategy, get_strategy, save_container, load_container, container_info, Comm, Loopback,
                  comm_unique_id, cp_als, tucker_cp, CpAlsResult, TuckerCpResult)

__all__ = ["KIND_N", "KIND_K", "PWC", "PWL", "DftService", "EmbeddedSpectrum", "GmresConfig", "GmresResult",
           "TuckerForm", "VieError", "apply_operator", "apply_operator_batch", "apply_system", "build_operator_spectra",
           "component_table", "gmres", "lib", "ncur", "tucker_compress", "RULE_ENERGY", "RULE_SIGMA_MAX",
           "DielectricMap", "Fields", "PlaneWave", "PostProcess", "VoxelGrid", "build_rhs", "postprocess",
           "recover_fields", "SolveReport", "solve_scene", "tucker_cp_form", "gmres_map", "ApplyTimings",
           "apply_operator_timed", "KIND_G", "QuadratureSpec", "assemble_defining_tensor", "assemble_operator",
           "self_static_term", "set_strategy", "get_strategy", "save_container", "load_container",
           "container_info", "Comm", "Loopback", "comm_unique_id", "cp_als", "tucker_cp",
           "CpAlsResult", "TuckerCpResult"]
