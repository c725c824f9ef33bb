"""B200-native data-parallel CNN training hot path of Omnivore (arXiv 1606.04487)."""
__version__ = "0.1.0"
