"""B200-native halftoning hot path of arXiv 2304.12152 (htlab drop-in).

Submodules mirror the reference package layout for the hot path:
  nn        PolicyNetwork / Parameter / Adam / cosine_lr  (htlab.nn)
  rl        infer_halftone / halftone / train_step / ...  (htlab.rl)
  metrics   MetricConfig / reward / delta_map             (htlab.metrics)
  spectral  ring_partition / anisotropy_loss(_backward)   (htlab.spectral)
  hvs       HVS stencil builders (host constants)         (htlab.hvs)
  imagecore Rng / gaussian_noise_map / random_crop        (htlab.imagecore)
All compute runs in the CUDA library csrc/libhtb200.so (sm_100a); importing a
compute entry point without it raises RuntimeError -- there is no CPU path.
"""

__version__ = "0.1.0"
