"""B200-native E-Tree / E-Forest ADC (arXiv 1509.05186) -- see DESIGN.md.

Submodules load lazily: ``synth`` (seeded inputs) needs neither torch nor the
CUDA library; ``api`` binds libetree.so (built by ``build.py``).
"""
__all__ = ["api", "synth", "build"]
