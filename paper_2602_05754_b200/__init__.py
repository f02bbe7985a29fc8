"""B200-native TimelyFreeze (arXiv 2602.05754) pipeline stage step with adaptive freezing."""
__version__ = "0.1.0"
