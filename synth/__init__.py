"""Seeded synthetic input generators (no method arithmetic; see kgsynth.py)."""
from .kgsynth import CONFIGS, GENERATOR_VERSION, Config, generate, generate_config, generate_se, sample_rows  # noqa: F401
