"""B200-native stochastic multiscale flux basis (Method S3) for sdmortar problems."""

__version__ = "0.1.0"
