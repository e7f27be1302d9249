"""ringpipe-b200: the Ouroboros delayed-gradient model-parallel training step
(arXiv 1909.06695) rebuilt B200-native behind the reference `ringpipe` API."""

__version__ = "0.1.0"
