"""BASELINE.json configurations 1-5 as data (SURVEY.md section 8 shape table).

Choices BASELINE.json leaves open are fixed here and
restated in DESIGN.md: noise "N(0, s)" is read as a standard deviation;
snapshot times are an inclusive linspace; rows are QoI-major; Omega_s is
distinct per subdomain (Philox counter = global subdomain id); config 3's
modes use nu = 0.01, t in [0, 10]; config 4 uses p = 16 (ell = 80) and the
blocked rule with the sketch-estimated error residual_fro / ||Y||_F.
"""
from __future__ import annotations

from dataclasses import dataclass

# field families (spidgpu_field_spec.kind); plain data, so the configs can be
# read without loading the CUDA library (bench.py's reference arm does)
FIELD_TGV4, FIELD_TGV5, FIELD_MULTIMODE = 0, 1, 2


@dataclass(frozen=True)
class SpidConfig:
    name: str
    kind: int            # field family (FIELD_*)
    grid: int            # N (per axis) of the whole grid
    block: int           # b (per axis) of a subdomain
    qois: int
    snapshots: int
    t_end: float
    nu: float
    sigma: float
    k: int
    p: int
    n_modes: int = 0
    kappa_max: float = 16.0
    mode_amp: float = 1e-2
    heavy_modes: int = 0
    heavy_kmin: float = 8.0
    adaptive: bool = False   # blocked rank rule (config 4)
    kstep: int = 8
    tol: float = 1e-3
    seed: int = 20210301
    per_gpu_subdomains: int | None = None  # weak scaling: subdomains per GPU
    note: str = ""

    @property
    def ell(self) -> int:
        return self.k + self.p

    @property
    def m(self) -> int:
        return self.qois * self.block ** 3

    @property
    def n(self) -> int:
        return self.snapshots

    @property
    def subdomains(self) -> int:
        return (self.grid // self.block) ** 3

    def field_spec(self):
        from . import _native as N

        return N.FieldSpec(self.kind, self.n_modes, self.grid, self.block, self.snapshots,
                           self.t_end, self.nu, self.sigma, self.kappa_max, self.mode_amp,
                           self.seed, self.heavy_modes, self.heavy_kmin)

    def field_dict(self) -> dict:
        """The same spec as plain values (oracle.port().field_generate)."""
        return dict(kind=self.kind, n_modes=self.n_modes, grid=self.grid, block=self.block,
                    snapshots=self.snapshots, t_end=self.t_end, nu=self.nu, sigma=self.sigma,
                    kappa_max=self.kappa_max, mode_amp=self.mode_amp, seed=self.seed,
                    heavy_modes=self.heavy_modes, heavy_kmin=self.heavy_kmin)

    def raw_bytes(self, subdomains: int | None = None) -> int:
        s = self.subdomains if subdomains is None else subdomains
        return 8 * self.m * self.n * s


CONFIGS = {
    # 1: analytic incompressible TGV, 32^3, 4 QoIs, 100 snapshots in [0,10],
    #    sigma 1e-8, 8 subdomains of 16^3, k=10, p=10
    "cfg1": SpidConfig("cfg1", FIELD_TGV4, 32, 16, 4, 100, 10.0, 0.01, 1e-8, 10, 10),
    # 2: compressible TGV at 128^3, 5 QoIs, 512 snapshots in [0,20], sigma 1e-6,
    #    64 subdomains of 32^3, k=20, p=10, single GPU
    "cfg2": SpidConfig("cfg2", FIELD_TGV5, 128, 32, 5, 512, 20.0, 0.01, 1e-6, 20, 10),
    # 3: TGV + 64 random Fourier modes, 5 QoIs, 256 snapshots, 128^3 per GPU
    #    (64 subdomains of 32^3 per GPU), k=32, p=16 -- weak scaling 1/2/4/8
    "cfg3": SpidConfig("cfg3", FIELD_MULTIMODE, 128, 32, 5, 256, 10.0, 0.01, 0.0, 32, 16,
                       n_modes=64, per_gpu_subdomains=64),
    # 4: config-3 field at 192^3 over 8 GPUs (216 subdomains), half with +256
    #    high-wavenumber modes; rank in steps of 8 up to 64 until the sketch
    #    error <= 1e-3 (ell = kmax + p = 80)
    "cfg4": SpidConfig("cfg4", FIELD_MULTIMODE, 192, 32, 5, 256, 10.0, 0.01, 0.0, 64, 16,
                       n_modes=64, heavy_modes=256, heavy_kmin=8.0, adaptive=True),
    # 5: config-3 field at 256^3 (512 subdomains, 64 per GPU over 8), k=32, p=16
    "cfg5": SpidConfig("cfg5", FIELD_MULTIMODE, 256, 32, 5, 256, 10.0, 0.01, 0.0, 32, 16,
                       n_modes=64, per_gpu_subdomains=64),
}


def weak_range(cfg: SpidConfig, rank: int, world: int) -> tuple[SpidConfig, int, int]:
    """Config 3 weak scaling: every GPU compresses 64 subdomains of 32^3 (128^3
    points). All world sizes draw them from the config-5 256^3 field, rank r
    taking global blocks [64r, 64r+64) in make_block_domains order, so at 8
    GPUs the run IS config 5 and at 1 GPU it is a 128^3-point slab of it."""
    if cfg.per_gpu_subdomains is None:
        raise ValueError(f"{cfg.name} is not a weak-scaling config")
    big = CONFIGS["cfg5"]
    per = cfg.per_gpu_subdomains
    if per * world > big.subdomains:
        raise ValueError("world too large for the 256^3 field")
    return big, rank * per, per
