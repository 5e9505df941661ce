"""Seeded synthetic inputs shared by `oracle/` (tests) and the CUDA path (bench/tests)."""
from .profiles import (CONFIGS, PLANNING_GRID_GPUS, PLANNING_GRID_LAYERS, PLANNING_GRID_NODES,
                       PLANNING_GRID_PAPER_S, Config, Profile, config_profiles, costs_profile, gpt_profile,
                       planning_grid_config, random_profile, unif6, uniform, splitmix64)

__all__ = ["CONFIGS", "PLANNING_GRID_GPUS", "PLANNING_GRID_LAYERS", "PLANNING_GRID_NODES", "PLANNING_GRID_PAPER_S",
           "planning_grid_config", "Config", "Profile", "config_profiles", "costs_profile", "gpt_profile",
           "random_profile", "unif6", "uniform", "splitmix64"]
