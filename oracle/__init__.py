"""CPU oracle for the B200 PIV generator -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (paper_2512_09664_b200/) imports this package;
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs use it, and only as the checker / the timed CPU
baseline -- never as a fallback for the GPU path.

Contents
  philox.py    numpy Philox4x32-10 (pinned to Random123 known-answer vectors and
               to NVIDIA's curand_Philox4x32_10 compiled for the host).
  generate.py  restatement of the seeding/advection path (reference
               particles.py:61-147, flowfield.py:207-232, config.py:139-146,
               raster.py:30-38) with the Philox draw layout of the B200 kernels;
               float64-exact parts are bit-identical to the GPU.
  render.py    restatement of splat/_native.splat_accumulate (_native.pyx:14-66),
               finalize (raster.py:154-161), quantize_u16 (export.py:19-20),
               the erf PSF and laser-sheet extensions, and the per-tile binning
               counts of the fused kernel.
  reference.py loader for the real reference package built into oracle/_ref
               (``oracle/build_ref.sh``), used to pin the restatement.
"""
