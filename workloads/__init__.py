"""Seeded synthetic inputs shared by `oracle/` (tests) and the CUDA path (bench/tests)."""
from .profiles import (CONFIGS, Config, Profile, config_profiles, costs_profile, gpt_profile,
                       random_profile, unif6, uniform, splitmix64)

__all__ = ["CONFIGS", "Config", "Profile", "config_profiles", "costs_profile", "gpt_profile",
           "random_profile", "unif6", "uniform", "splitmix64"]
