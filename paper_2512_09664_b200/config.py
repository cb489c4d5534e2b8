"""Generation recipe: the reference's YAML schema plus B200 extensions.

Drop-in for the reference ``pivgen.config`` (config.py:1-462): same keys,
defaults, validation messages (``ConfigError`` names the offending field,
config.py:149-241), unknown-key rejection (config.py:350-352) and the
``render_config`` / ``parse_config`` round trip (config.py:404-457).

Differences, all opt-in so a reference document means reference behaviour:
  * ``device`` accepts ``cuda`` / ``cuda:N`` (default ``cuda``); the legacy
    value ``cpu`` is accepted and means "the current CUDA device" -- there is
    no CPU generation path in this package.
  * ``psf``: ``point`` (reference Eq. (1) at pixel centres) or ``erf``
    (pixel-area integration).
  * ``output_dtype``: ``float32`` (reference) or ``uint16`` (band-kernel
    ``quantize_u16``, export.py:19-20, bit-exact).
  * ``rng``: ``philox`` (the B200 generator's Philox4x32-10 streams) or
    ``splitmix64`` (the reference's own rng.py streams: particle arrays
    bit-identical to the reference, images within 1e-5; point PSF only).
  * ``laser_sheet``: out-of-plane position and the Remark-1 intensity profile
    I0(z) = q exp(-(1/sqrt(2 pi)) |2 z^2 / dZ0^2|^s).

The schema is expressed once as a table of ``_Field`` entries that drive
parsing, validation and rendering.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, fields, replace
from typing import Any, Callable

import yaml

RHO_LIMIT = 1.0 - 1e-3

OUTPUT_FORMATS = ("png16", "raw_f32")
SOURCE_FORMATS = ("flo", "npy_xyuv", "hdf5", "function")
PSF_KINDS = ("point", "erf")
OUTPUT_DTYPES = ("float32", "uint16")
RNG_KINDS = ("philox", "splitmix64")   # splitmix64: the reference's rng.py streams

_SUFFIX_FORMAT = (
    (".flo", "flo"),
    (".npy", "npy_xyuv"),
    (".h5", "hdf5"),
    (".hdf5", "hdf5"),
)


class ConfigError(ValueError):
    """Invalid configuration document or field value."""


def _fail(name: str, message: str) -> None:
    raise ConfigError(f"{name}: {message}")


# ---------------------------------------------------------------------------
# Nested records
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class FlowSource:
    """A flow file path or a registered flow function (config.py:38-66)."""

    path: str | None = None
    format: str | None = None
    function: str | None = None
    u_dataset: str = "u"
    v_dataset: str = "v"
    scale: float = 1.0

    def resolved_format(self) -> str:
        if self.format is not None:
            return self.format
        if self.function is not None:
            return "function"
        lowered = (self.path or "").lower()
        for suffix, fmt in _SUFFIX_FORMAT:
            if lowered.endswith(suffix):
                return fmt
        raise ConfigError(f"flow_sources: cannot infer format from path {self.path!r}; "
                          "set 'format' explicitly")


@dataclass(frozen=True)
class NoiseConfig:
    background_offset: float = 0.0
    gaussian_std: float = 0.0

    @property
    def enabled(self) -> bool:
        return self.background_offset != 0.0 or self.gaussian_std != 0.0


@dataclass(frozen=True)
class OutputConfig:
    format: str = "png16"
    directory: str = "out"


@dataclass(frozen=True)
class LaserSheetConfig:
    """Out-of-plane seeding + laser-sheet intensity.

    z1 ~ U[z_range]; z2 = z1 + out_of_plane; peak intensity of frame k is the
    sampled I0 times I0(z_k) = efficiency * exp(-(1/sqrt(2 pi)) |2 z^2 / thickness^2|^shape).
    z_range defaults to [-thickness, thickness].
    """

    thickness: float = 1.0
    shape: float = 2.0
    efficiency: float = 1.0
    z_range: tuple[float, float] | None = None
    out_of_plane: float = 0.0

    def resolved_z_range(self) -> tuple[float, float]:
        if self.z_range is not None:
            return (float(self.z_range[0]), float(self.z_range[1]))
        return (-self.thickness, self.thickness)


# ---------------------------------------------------------------------------
# The configuration
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class GeneratorConfig:
    """Validated, immutable generation recipe (fields as config.py:87-108)."""

    image_height: int = 512
    image_width: int = 512
    batch_size: int = 64
    flow_fields_per_batch: int = 1
    batches_per_flow_field: int = 1
    seeding_density_range: tuple[float, float] = (0.06, 0.06)
    diameter_range: tuple[float, float] = (0.8, 1.2)
    peak_intensity_range: tuple[float, float] = (1.0, 1.0)
    rho_range: tuple[float, float] = (0.0, 0.0)
    frame2_sigma_std: float = 0.0
    frame2_rho_std: float = 0.0
    frame2_intensity_std: float = 0.0
    hide_probability: float = 0.0
    noise: NoiseConfig = field(default_factory=NoiseConfig)
    target_histogram: tuple[float, ...] | None = None
    flow_sources: tuple[FlowSource, ...] = ()
    seed: int = 0
    threads: int = 0
    output: OutputConfig = field(default_factory=OutputConfig)
    device: str = "cuda"
    diameter_sigma_ratio: float = 4.0
    patch_multiplier: float = 3.0
    # --- B200 extensions ---
    psf: str = "point"
    output_dtype: str = "float32"
    rng: str = "philox"
    laser_sheet: LaserSheetConfig | None = None

    def __post_init__(self) -> None:
        _canonicalize(self)
        validate_config(self)

    @property
    def pairs_per_field(self) -> int:
        return self.batch_size // self.flow_fields_per_batch

    def particle_capacity(self) -> int:
        """N = ceil(ppp_max * H * W) with a 9-digit guard (config.py:139-146)."""
        n = self.seeding_density_range[1] * self.image_height * self.image_width
        return math.ceil(round(n, 9))

    @property
    def device_index(self) -> int | None:
        """CUDA ordinal requested by ``device`` (None = current device)."""
        if ":" in self.device:
            return int(self.device.split(":", 1)[1])
        return None


_RANGE_FIELDS = ("seeding_density_range", "diameter_range", "peak_intensity_range", "rho_range")
_FLOAT_FIELDS = ("frame2_sigma_std", "frame2_rho_std", "frame2_intensity_std",
                 "hide_probability", "diameter_sigma_ratio", "patch_multiplier")


def _as_float_if_int(x: Any) -> Any:
    return float(x) if isinstance(x, int) and not isinstance(x, bool) else x


def _canonicalize(cfg: GeneratorConfig) -> None:
    set_ = object.__setattr__
    for name in _RANGE_FIELDS:
        value = getattr(cfg, name)
        if isinstance(value, (list, tuple)) and len(value) == 2:
            set_(cfg, name, (_as_float_if_int(value[0]), _as_float_if_int(value[1])))
    for name in _FLOAT_FIELDS:
        set_(cfg, name, _as_float_if_int(getattr(cfg, name)))
    if cfg.target_histogram is not None:
        set_(cfg, "target_histogram", tuple(_as_float_if_int(x) for x in cfg.target_histogram))
    if not isinstance(cfg.flow_sources, tuple):
        set_(cfg, "flow_sources", tuple(cfg.flow_sources))
    if isinstance(cfg.laser_sheet, dict):
        set_(cfg, "laser_sheet", _parse_laser(cfg.laser_sheet))


# ---------------------------------------------------------------------------
# Validation (total: raises ConfigError naming the field)
# ---------------------------------------------------------------------------

def _check_range(cfg: GeneratorConfig, name: str, lo_bound: float, hi_bound: float,
                 open_lo: bool = False, open_hi: bool = False) -> None:
    value = getattr(cfg, name)
    if not (isinstance(value, tuple) and len(value) == 2):
        _fail(name, "must be a [min, max] pair")
    lo, hi = value
    if not all(isinstance(x, float) and math.isfinite(x) for x in value):
        _fail(name, "bounds must be finite numbers")
    if lo > hi:
        _fail(name, f"min {lo} exceeds max {hi}")
    if (lo <= lo_bound) if open_lo else (lo < lo_bound):
        _fail(name, f"min {lo} out of bounds")
    if (hi >= hi_bound) if open_hi else (hi > hi_bound):
        _fail(name, f"max {hi} out of bounds")


def _positive_int(cfg: GeneratorConfig, name: str) -> None:
    value = getattr(cfg, name)
    if not (isinstance(value, int) and not isinstance(value, bool) and value > 0):
        _fail(name, f"must be a positive integer, got {value!r}")


def validate_config(cfg: GeneratorConfig) -> None:
    for name in ("image_height", "image_width", "batch_size", "flow_fields_per_batch",
                 "batches_per_flow_field"):
        _positive_int(cfg, name)
    if cfg.batch_size % cfg.flow_fields_per_batch:
        _fail("flow_fields_per_batch",
              f"must divide batch_size ({cfg.flow_fields_per_batch} does not divide "
              f"{cfg.batch_size})")
    if cfg.image_height >= 16384 or cfg.image_width >= 16384:
        _fail("image_height" if cfg.image_height >= 16384 else "image_width",
              "must be below 16384 pixels")

    _check_range(cfg, "seeding_density_range", 0.0, math.inf, open_lo=True, open_hi=True)
    _check_range(cfg, "diameter_range", 0.0, math.inf, open_lo=True, open_hi=True)
    _check_range(cfg, "peak_intensity_range", 0.0, 1.0)
    _check_range(cfg, "rho_range", -RHO_LIMIT, RHO_LIMIT)
    if cfg.particle_capacity() < 1:
        _fail("seeding_density_range",
              "ppp_max * height * width must allow at least one particle")
    if cfg.particle_capacity() >= 2 ** 31:
        _fail("seeding_density_range", "particle capacity must be below 2^31")

    for name in ("frame2_sigma_std", "frame2_rho_std", "frame2_intensity_std"):
        value = getattr(cfg, name)
        if not (isinstance(value, float) and math.isfinite(value) and value >= 0.0):
            _fail(name, f"must be a non-negative number, got {value!r}")
    if not (isinstance(cfg.hide_probability, float) and 0.0 <= cfg.hide_probability < 1.0):
        _fail("hide_probability", f"must lie in [0, 1), got {cfg.hide_probability!r}")

    if not isinstance(cfg.noise, NoiseConfig):
        _fail("noise", "must be a mapping")
    if not 0.0 <= cfg.noise.background_offset < 1.0:
        _fail("noise.background_offset",
              f"must lie in [0, 1), got {cfg.noise.background_offset!r}")
    if not cfg.noise.gaussian_std >= 0.0:
        _fail("noise.gaussian_std", f"must be non-negative, got {cfg.noise.gaussian_std!r}")

    if cfg.target_histogram is not None:
        hist = cfg.target_histogram
        if len(hist) != 256:
            _fail("target_histogram", f"must have exactly 256 bins, got {len(hist)}")
        if not all(math.isfinite(x) and x >= 0.0 for x in hist):
            _fail("target_histogram", "bins must be finite and non-negative")
        if not sum(hist) > 0.0:
            _fail("target_histogram", "must have a positive sum")

    for i, src in enumerate(cfg.flow_sources):
        name = f"flow_sources[{i}]"
        if not isinstance(src, FlowSource):
            _fail(name, "must be a mapping")
        if (src.path is None) == (src.function is None):
            _fail(name, "exactly one of 'path' or 'function' is required")
        if src.format is not None:
            if src.format not in SOURCE_FORMATS:
                _fail(name, f"unknown format {src.format!r}; expected one of {SOURCE_FORMATS}")
            if (src.format == "function") != (src.function is not None):
                _fail(name, "'function' entries must use format 'function' and vice versa")
        src.resolved_format()
        if not (math.isfinite(src.scale) and src.scale != 0.0):
            _fail(f"{name}.scale", f"must be finite and non-zero, got {src.scale!r}")

    if not (isinstance(cfg.seed, int) and not isinstance(cfg.seed, bool) and 0 <= cfg.seed < 2 ** 64):
        _fail("seed", f"must be a 64-bit unsigned integer, got {cfg.seed!r}")
    if not (isinstance(cfg.threads, int) and cfg.threads >= 0):
        _fail("threads", f"must be 0 (auto) or a positive integer, got {cfg.threads!r}")
    if cfg.output.format not in OUTPUT_FORMATS:
        _fail("output.format", f"must be one of {OUTPUT_FORMATS}, got {cfg.output.format!r}")
    if not cfg.output.directory:
        _fail("output.directory", "must be non-empty")

    dev = cfg.device
    ok_dev = dev in ("cpu", "cuda") or (dev.startswith("cuda:") and dev[5:].isdigit())
    if not (isinstance(dev, str) and ok_dev):
        _fail("device", f"must be 'cuda', 'cuda:N' (or legacy 'cpu'), got {dev!r}")

    for name in ("diameter_sigma_ratio", "patch_multiplier"):
        value = getattr(cfg, name)
        if not (isinstance(value, float) and math.isfinite(value) and value > 0.0):
            _fail(name, f"must be a positive number, got {value!r}")

    if cfg.psf not in PSF_KINDS:
        _fail("psf", f"must be one of {PSF_KINDS}, got {cfg.psf!r}")
    if cfg.output_dtype not in OUTPUT_DTYPES:
        _fail("output_dtype", f"must be one of {OUTPUT_DTYPES}, got {cfg.output_dtype!r}")
    if cfg.rng not in RNG_KINDS:
        _fail("rng", f"must be one of {RNG_KINDS}, got {cfg.rng!r}")
    if cfg.rng == "splitmix64" and (cfg.psf != "point" or cfg.laser_sheet is not None):
        _fail("rng", "splitmix64 (reference RNG) mode renders the reference model: point PSF, no laser sheet")
    if cfg.laser_sheet is not None:
        ls = cfg.laser_sheet
        if not isinstance(ls, LaserSheetConfig):
            _fail("laser_sheet", "must be a mapping")
        if not (math.isfinite(ls.thickness) and ls.thickness > 0.0):
            _fail("laser_sheet.thickness", f"must be positive, got {ls.thickness!r}")
        if not (math.isfinite(ls.shape) and ls.shape > 0.0):
            _fail("laser_sheet.shape", f"must be positive, got {ls.shape!r}")
        if not (0.0 < ls.efficiency <= 1.0):
            _fail("laser_sheet.efficiency", f"must lie in (0, 1], got {ls.efficiency!r}")
        zlo, zhi = ls.resolved_z_range()
        if not (math.isfinite(zlo) and math.isfinite(zhi) and zlo <= zhi):
            _fail("laser_sheet.z_range", f"must be a finite [min, max] pair, got {ls.z_range!r}")
        if not math.isfinite(ls.out_of_plane):
            _fail("laser_sheet.out_of_plane", "must be finite")


def default_config() -> GeneratorConfig:
    return GeneratorConfig()


# ---------------------------------------------------------------------------
# Parsing / rendering, driven by one field table
# ---------------------------------------------------------------------------

def _p_int(value: Any, name: str) -> int:
    if isinstance(value, bool) or not isinstance(value, int):
        raise ConfigError(f"{name}: expected an integer, got {value!r}")
    return value


def _p_float(value: Any, name: str) -> float:
    if isinstance(value, bool) or not isinstance(value, (int, float)):
        raise ConfigError(f"{name}: expected a number, got {value!r}")
    return float(value)


def _p_str(value: Any, name: str) -> str:
    if not isinstance(value, str):
        raise ConfigError(f"{name}: expected a string, got {value!r}")
    return value


def _p_pair(value: Any, name: str) -> tuple[float, float]:
    if not isinstance(value, (list, tuple)) or len(value) != 2:
        raise ConfigError(f"{name}: expected a [min, max] pair, got {value!r}")
    return (_p_float(value[0], name), _p_float(value[1], name))


def _p_mapping(value: Any, name: str, allowed: set[str]) -> dict:
    if not isinstance(value, dict):
        raise ConfigError(f"{name}: expected a mapping, got {value!r}")
    extra = set(value) - allowed
    if extra:
        raise ConfigError(f"{name}: unknown key(s) {sorted(extra)}")
    return value


def _p_noise(value: Any, name: str) -> NoiseConfig:
    data = _p_mapping(value, name, {"background_offset", "gaussian_std"})
    return NoiseConfig(
        background_offset=_p_float(data.get("background_offset", 0.0), f"{name}.background_offset"),
        gaussian_std=_p_float(data.get("gaussian_std", 0.0), f"{name}.gaussian_std"))


def _p_output(value: Any, name: str) -> OutputConfig:
    data = _p_mapping(value, name, {"format", "directory"})
    return OutputConfig(format=_p_str(data.get("format", "png16"), f"{name}.format"),
                        directory=_p_str(data.get("directory", "out"), f"{name}.directory"))


def _p_histogram(value: Any, name: str):
    if value in (None, []):
        return None
    if not isinstance(value, list):
        raise ConfigError(f"{name}: expected a list of 256 bins, got {value!r}")
    return tuple(_p_float(x, name) for x in value)


_SOURCE_KEYS = {"path": _p_str, "format": _p_str, "function": _p_str,
                "u_dataset": _p_str, "v_dataset": _p_str, "scale": _p_float}


def _p_sources(value: Any, name: str) -> tuple[FlowSource, ...]:
    if not isinstance(value, list):
        raise ConfigError(f"{name}: expected a list, got {value!r}")
    out = []
    for i, entry in enumerate(value):
        ename = f"{name}[{i}]"
        data = _p_mapping(entry, ename, set(_SOURCE_KEYS))
        if "path" not in data and "function" not in data:
            raise ConfigError(f"{ename}: requires 'path' or 'function'")
        out.append(FlowSource(**{k: p(data[k], f"{ename}.{k}") for k, p in _SOURCE_KEYS.items()
                                 if k in data}))
    return tuple(out)


def _parse_laser(data: dict, name: str = "laser_sheet") -> LaserSheetConfig:
    data = _p_mapping(data, name, {"thickness", "shape", "efficiency", "z_range", "out_of_plane"})
    kw: dict[str, Any] = {}
    for key in ("thickness", "shape", "efficiency", "out_of_plane"):
        if key in data:
            kw[key] = _p_float(data[key], f"{name}.{key}")
    if data.get("z_range") is not None:
        kw["z_range"] = _p_pair(data["z_range"], f"{name}.z_range")
    return LaserSheetConfig(**kw)


def _p_laser(value: Any, name: str):
    if value is None:
        return None
    return _parse_laser(value, name)


def _r_identity(v):
    return v


def _r_list(v):
    return list(v)


def _r_noise(v: NoiseConfig):
    return {"background_offset": v.background_offset, "gaussian_std": v.gaussian_std}


def _r_output(v: OutputConfig):
    return {"format": v.format, "directory": v.directory}


def _r_sources(v):
    entries = []
    for src in v:
        e: dict[str, Any] = {}
        if src.path is not None:
            e["path"] = src.path
        if src.function is not None:
            e["function"] = src.function
        if src.format is not None:
            e["format"] = src.format
        if src.u_dataset != "u":
            e["u_dataset"] = src.u_dataset
        if src.v_dataset != "v":
            e["v_dataset"] = src.v_dataset
        if src.scale != 1.0:
            e["scale"] = src.scale
        entries.append(e)
    return entries


def _r_laser(v: LaserSheetConfig | None):
    if v is None:
        return None
    out = {"thickness": v.thickness, "shape": v.shape, "efficiency": v.efficiency,
           "out_of_plane": v.out_of_plane}
    if v.z_range is not None:
        out["z_range"] = list(v.z_range)
    return out


@dataclass(frozen=True)
class _Field:
    name: str
    parse: Callable[[Any, str], Any]
    render: Callable[[Any], Any] = _r_identity
    optional: bool = False     # rendered only when not None / non-empty


# Order = rendered document order (mirrors config.py:409-444 then extensions).
_SCHEMA: tuple[_Field, ...] = (
    _Field("image_height", _p_int),
    _Field("image_width", _p_int),
    _Field("batch_size", _p_int),
    _Field("flow_fields_per_batch", _p_int),
    _Field("batches_per_flow_field", _p_int),
    _Field("seeding_density_range", _p_pair, _r_list),
    _Field("diameter_range", _p_pair, _r_list),
    _Field("peak_intensity_range", _p_pair, _r_list),
    _Field("rho_range", _p_pair, _r_list),
    _Field("frame2_sigma_std", _p_float),
    _Field("frame2_rho_std", _p_float),
    _Field("frame2_intensity_std", _p_float),
    _Field("hide_probability", _p_float),
    _Field("noise", _p_noise, _r_noise),
    _Field("seed", _p_int),
    _Field("threads", _p_int),
    _Field("output", _p_output, _r_output),
    _Field("device", _p_str),
    _Field("diameter_sigma_ratio", _p_float),
    _Field("patch_multiplier", _p_float),
    _Field("psf", _p_str),
    _Field("output_dtype", _p_str),
    _Field("rng", _p_str),
    _Field("target_histogram", _p_histogram, _r_list, optional=True),
    _Field("flow_sources", _p_sources, _r_sources, optional=True),
    _Field("laser_sheet", _p_laser, _r_laser, optional=True),
)
_KNOWN = {f.name for f in _SCHEMA}


def parse_config(text: str) -> GeneratorConfig:
    """YAML document -> validated GeneratorConfig (config.py:332-396 semantics)."""
    try:
        data = yaml.safe_load(text)
    except yaml.YAMLError as exc:
        mark = getattr(exc, "problem_mark", None)
        where = f" at line {mark.line + 1}" if mark is not None else ""
        raise ConfigError(f"syntax error{where}: {exc}") from exc
    if data is None:
        data = {}
    if not isinstance(data, dict):
        raise ConfigError("document must be a key/value mapping")
    unknown = set(data) - _KNOWN
    if unknown:
        raise ConfigError(f"unknown key(s): {sorted(unknown)}")
    kwargs = {f.name: f.parse(data[f.name], f.name) for f in _SCHEMA if f.name in data}
    return GeneratorConfig(**kwargs)


def load_config(path: str) -> GeneratorConfig:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_config(fh.read())


def render_config(cfg: GeneratorConfig) -> str:
    """Inverse of parse_config: ``parse_config(render_config(c)) == c``."""
    doc: dict[str, Any] = {}
    for f in _SCHEMA:
        value = getattr(cfg, f.name)
        if f.optional and not value:
            continue
        doc[f.name] = f.render(value)
    return yaml.safe_dump(doc, sort_keys=False, default_flow_style=None)


def with_updates(cfg: GeneratorConfig, **changes: Any) -> GeneratorConfig:
    """dataclasses.replace that re-runs validation."""
    return replace(cfg, **changes)


def config_fields() -> tuple[str, ...]:
    return tuple(f.name for f in fields(GeneratorConfig))
