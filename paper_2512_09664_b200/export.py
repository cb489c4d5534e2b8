"""Dataset export: the reference's on-disk format,
written while the GPU generates the next batch.

Formats (reference export.py:1-52, cli.py:51-131):
* png16: 16-bit grayscale PNG of rint(clip(v, 0, 1) * 65535) (the uint16
  quantisation runs on the GPU, bit-identical to export.quantize_u16);
* raw_f32: int32 height, int32 width (little endian), then row-major
  little-endian float32 intensities;
* per pair: ``pair_{batch:06d}_{pair:04d}_a.{png|raw}``, ``..._b.{ext}``,
  ``..._flow.flo`` (Middlebury .flo); per batch ``params_{batch:06d}.json``
  (schema 1: per-pair density, counts and diameter / intensity / rho ranges,
  patch side), sorted keys, indent 1, trailing newline.

The image stacks leave the device through pinned host buffers on a side
stream (``non_blocking`` copies, one event per batch); a writer thread turns
them into files while the Sampler renders the next batch. A batch whose
write fails is removed so the tree stays consistent (cli.py:107-116).
"""

from __future__ import annotations

import json
import os
import queue
import struct
import threading
import time

import numpy as np
import torch

from .flowfield import write_flo_file
from .raster import patch_side

PARAMS_SCHEMA_VERSION = 1          # reference cli.py:35
_RAW_HEADER = struct.Struct("<ii")


def quantize_u16_host(img: np.ndarray) -> np.ndarray:
    """rint(clip(x, 0, 1) * 65535) in float32 (export.py:19-20) for host arrays."""
    x = np.clip(np.asarray(img, dtype=np.float32), np.float32(0.0), np.float32(1.0))
    return np.rint(x * np.float32(65535.0)).astype(np.uint16)


def write_png16(path: str, img: np.ndarray) -> None:
    """16-bit grayscale PNG (export.py:23-25). Accepts uint16 levels or float
    intensities in [0, 1]."""
    from PIL import Image

    a = np.asarray(img)
    data = a if a.dtype == np.uint16 else quantize_u16_host(a)
    im = Image.fromarray(np.ascontiguousarray(data))   # uint16 -> mode "I;16"
    im.save(path, format="PNG")


def read_png16(path: str) -> np.ndarray:
    from PIL import Image

    with Image.open(path) as im:
        data = np.asarray(im, dtype=np.uint16)
    return data.astype(np.float32) / 65535.0


def write_raw_f32(path: str, img: np.ndarray) -> None:
    arr = np.ascontiguousarray(img, dtype="<f4")
    with open(path, "wb") as fh:
        fh.write(_RAW_HEADER.pack(arr.shape[0], arr.shape[1]))
        fh.write(arr.tobytes())


def read_raw_f32(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < _RAW_HEADER.size:
        raise ValueError(f"raw_f32: truncated header in {path}")
    height, width = _RAW_HEADER.unpack_from(data)
    if height <= 0 or width <= 0 or len(data) != _RAW_HEADER.size + 4 * height * width:
        raise ValueError(f"raw_f32: corrupt payload in {path}")
    return np.frombuffer(data, dtype="<f4", offset=_RAW_HEADER.size).reshape(height, width).copy()


def pair_paths(out_dir: str, ext: str, batch: int, pair: int) -> list[str]:
    stem = os.path.join(out_dir, f"pair_{batch:06d}_{pair:04d}")
    return [f"{stem}_a.{ext}", f"{stem}_b.{ext}", f"{stem}_flow.flo"]


def _pair_start(batch) -> int:
    """Global index of the batch's first pair (a shard under torch.distributed)."""
    pr = getattr(batch, "pair_range", None)
    return pr.start if pr is not None and len(pr) else 0


def _is_shard(cfg, batch) -> bool:
    pr = getattr(batch, "pair_range", None)
    return pr is not None and len(pr) > 0 and len(pr) != cfg.batch_size


def sidecar(cfg, batch) -> dict:
    """Per-batch parameter sidecar (schema 1, reference cli.py:62-88); pair
    indices are global (a shard's pairs keep their place in the batch)."""
    pairs = []
    start = _pair_start(batch)
    for i, p in enumerate(batch.params):
        m = int(p.active_count)
        d = np.asarray(p.diameters)[:m]
        i0 = np.asarray(p.peak_intensities)[:m]
        rho = np.asarray(p.rhos)[:m]
        d_max = float(d.max()) if m else cfg.diameter_range[1]
        pairs.append({
            "pair_index": start + i,
            "seeding_density": float(p.seeding_density),
            "active_count": m,
            "allocated_count": int(np.asarray(p.diameters).shape[0]),
            "diameter_min": float(d.min()) if m else None,
            "diameter_max": float(d.max()) if m else None,
            "peak_intensity_min": float(i0.min()) if m else None,
            "peak_intensity_max": float(i0.max()) if m else None,
            "rho_min": float(rho.min()) if m else None,
            "rho_max": float(rho.max()) if m else None,
            "patch_side": patch_side(d_max, cfg.patch_multiplier),
        })
    return {"schema_version": PARAMS_SCHEMA_VERSION, "batch_index": int(batch.batch_index),
            "image_height": cfg.image_height, "image_width": cfg.image_width, "pairs": pairs}


class DatasetWriter:
    """Asynchronous writer: ``submit(batch)`` starts the D2H copies of the
    batch's images (uint16 levels for png16, float32 for raw_f32) into pinned
    buffers on a side stream and returns; a thread writes the files once the
    copies have landed. ``close()`` drains and re-raises the first error."""

    def __init__(self, cfg, out_dir: str, depth: int = 2):
        fmt = cfg.output.format
        if fmt not in ("png16", "raw_f32"):
            raise ValueError(f"unknown output format {fmt!r}")
        self.cfg = cfg
        self.out_dir = out_dir
        self.png = fmt == "png16"
        self.ext = "png" if self.png else "raw"
        os.makedirs(out_dir, exist_ok=True)
        if not os.access(out_dir, os.W_OK):
            raise OSError(f"output directory {out_dir!r} is not writable")
        self._q: queue.Queue = queue.Queue(maxsize=max(1, depth))
        self._err: BaseException | None = None
        self._stream = None
        self.written = 0
        self._thread = threading.Thread(target=self._run, name="pgb-export", daemon=True)
        self._thread.start()

    def _host_copy(self, stack: torch.Tensor):
        if not stack.is_cuda:
            return stack.numpy(), None
        if self.png and stack.dtype != torch.uint16:
            from .raster import quantize_u16

            stack = quantize_u16(stack)
        elif not self.png and stack.dtype != torch.float32:
            stack = stack.float() / 65535.0
        if self._stream is None:
            self._stream = torch.cuda.Stream(device=stack.device)
        host = torch.empty(stack.shape, dtype=stack.dtype, pin_memory=True)
        self._stream.wait_stream(torch.cuda.current_stream(stack.device))
        with torch.cuda.stream(self._stream):
            host.copy_(stack, non_blocking=True)
            stack.record_stream(self._stream)
            ev = torch.cuda.Event()
            ev.record(self._stream)
        return host, ev

    def submit(self, batch) -> None:
        if self._err is not None:
            raise self._err
        h1, e1 = self._host_copy(batch.images1)
        h2, e2 = self._host_copy(batch.images2)
        # the sidecar and flows need host data anyway: materialise them here
        meta = sidecar(self.cfg, batch)
        flows = list(batch.flow_fields)
        pr = getattr(batch, "pair_range", None)
        part = (pr.start, pr.stop) if _is_shard(self.cfg, batch) else None
        self._q.put((batch.batch_index, h1, h2, (e1, e2), flows, meta, _pair_start(batch), part))

    def _run(self) -> None:
        writer = write_png16 if self.png else write_raw_f32
        while True:
            item = self._q.get()
            if item is None:
                return
            if self._err is not None:
                continue
            b, h1, h2, events, flows, meta, start, part = item
            written: list[str] = []
            try:
                for ev in events:
                    if ev is not None:
                        ev.synchronize()
                a1 = h1.numpy() if isinstance(h1, torch.Tensor) else h1
                a2 = h2.numpy() if isinstance(h2, torch.Tensor) else h2
                for i in range(a1.shape[0]):
                    pa, pb, pf = pair_paths(self.out_dir, self.ext, b, start + i)
                    writer(pa, a1[i])
                    written.append(pa)
                    writer(pb, a2[i])
                    written.append(pb)
                    if flows:
                        write_flo_file(pf, flows[i])
                        written.append(pf)
                # a shard writes its part of the sidecar; merge_sidecars() joins them
                name = f"params_{b:06d}.json" if part is None else f"params_{b:06d}.part{part[0]:05d}-{part[1]:05d}.json"
                path = os.path.join(self.out_dir, name)
                with open(path, "w", encoding="utf-8") as fh:
                    json.dump(meta, fh, sort_keys=True, indent=1)
                    fh.write("\n")
                written.append(path)
                self.written += a1.shape[0]
            except BaseException as e:  # keep the tree consistent, report on the next call
                for path in written:
                    try:
                        os.remove(path)
                    except OSError:
                        pass
                self._err = e

    def close(self) -> None:
        if self._thread.is_alive():
            self._q.put(None)
            self._thread.join()
        if self._err is not None:
            raise self._err

    def __enter__(self) -> "DatasetWriter":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def merge_sidecars(out_dir: str) -> int:
    """Join the per-shard sidecar parts of every batch into ``params_<b>.json``
    (pairs ordered by global index) and delete the parts. Returns the number
    of merged batches."""
    import glob
    import re

    groups: dict[str, list[str]] = {}
    for path in glob.glob(os.path.join(out_dir, "params_*.part*.json")):
        m = re.match(r"(params_\d+)\.part\d+-\d+\.json$", os.path.basename(path))
        if m:
            groups.setdefault(m.group(1), []).append(path)
    for stem, parts in groups.items():
        docs = []
        for path in sorted(parts):
            with open(path, encoding="utf-8") as fh:
                docs.append(json.load(fh))
        merged = dict(docs[0])
        merged["pairs"] = sorted((p for d in docs for p in d["pairs"]), key=lambda p: p["pair_index"])
        with open(os.path.join(out_dir, stem + ".json"), "w", encoding="utf-8") as fh:
            json.dump(merged, fh, sort_keys=True, indent=1)
            fh.write("\n")
        for path in parts:
            os.remove(path)
    return len(groups)


def generate_dataset(cfg, batches: int, out_dir: str, start_batch: int = 0) -> dict:
    """``pivgen generate`` (reference cli.py:91-131): ``batches`` batches into
    ``out_dir`` in the reference layout. Returns counts and wall time.

    Under torch.distributed every rank writes its shard of each batch (global
    pair indices in file names and sidecar); after a barrier rank 0 merges the
    sidecar parts. ``pairs`` counts this rank's pairs, ``pairs_total`` the job's."""
    from .pipeline import Sampler

    t0 = time.perf_counter()
    total = 0
    with DatasetWriter(cfg, out_dir) as w, Sampler(cfg, start_batch=start_batch, max_batches=batches) as s:
        shard = len(s.pair_range)
        for batch in s:
            w.submit(batch)
            total += shard
    dist_on = torch.distributed.is_available() and torch.distributed.is_initialized()
    if dist_on and torch.distributed.get_world_size() > 1:
        torch.distributed.barrier()
        if torch.distributed.get_rank() == 0:
            merge_sidecars(out_dir)
        torch.distributed.barrier()
    return {"pairs": total, "pairs_total": cfg.batch_size * batches, "batches": batches, "dir": out_dir,
            "seconds": time.perf_counter() - t0}
