"""Counter-based synthetic event generators for configs C1..C5 (numpy).

INPUT-GENERATION module: the recipe of SURVEY.md §8d ("Common generator
recipe") made concrete.  The same recipe is implemented independently in CUDA
(gxin/gen_cuda.cu -> libgxgen.so) for the large batches bench.py times; a GPU
test checks the two byte for byte.  Every field of event i is a pure function
of (seed, config, i, n_total), so any shard [i0, i0+n) of a batch can be
generated on its own (multi-GPU sharding).

    mix64  = SplitMix64 finalizer
    rnd(seed, stream, j) = mix64((seed ^ stream*0xD1B54A32D192ED03) + j*0x9E3779B97F4A7C15)
    record fields use j = rec = i >> 5, lane fields use j = i, lane_id = i & 31
    skewed draws: u64 threshold tables t_k = floor(CDF_k * 2^64) (last = 2^64-1),
                  sample = #{k : t_k <= u}, clamped to K-1  (bit-identical everywhere)

The shapes follow the paper's workloads: Fig 1 access patterns (PAPER.md:81-86:
MoE prefill periodic-sequential, decode sparse-random; faiss build sequential,
query random), Fig 2's SM/warp imbalance, the IVF4096 layout
of the Faiss experiment.
"""
from __future__ import annotations

import functools

import numpy as np

M64 = (1 << 64) - 1
C_STREAM = 0xD1B54A32D192ED03
C_GOLD = 0x9E3779B97F4A7C15

EVENT_DTYPE = np.dtype([("addr", "<u8"), ("ts", "<u8"), ("hook", "<u4"), ("block_id", "<u4"),
                        ("sm_id", "<u2"), ("warp_id", "u1"), ("lane_id", "u1"), ("size", "<u4")])
assert EVENT_DTYPE.itemsize == 32

CONFIGS = ("C1", "C2", "C3", "C4", "C5")
CONFIG_ID = {c: k + 1 for k, c in enumerate(CONFIGS)}

# C3 address space: 4 GiB = 2^20 pages; weights = 24 experts x 32768 pages
NPAGES = 1 << 20
NWEIGHT = 24 * 32768
PERM_A, PERM_B = 500009, 12345          # bijection on [0, NWEIGHT): 500009 is coprime to 2^18*3
# C4 layout (Faiss IVF4096,Flat shape)
NLISTS = 4096
CENTROID_BYTES = 2 << 20
QUERY_RECS = 64 + 16 * 32               # 64 centroid records + nprobe=16 lists x 32 records
LAYOUT_SEED = 0x1F4096


def _u64(x):
    return np.asarray(x, dtype=np.uint64)


def mix64(x):
    x = _u64(x).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def rnd(seed: int, stream: int, j):
    base = np.uint64((seed ^ ((stream * C_STREAM) & M64)) & M64)
    with np.errstate(over="ignore"):
        return mix64(base + _u64(j) * np.uint64(C_GOLD))


def quantize_cdf(weights) -> np.ndarray:
    """u64 threshold table from (unnormalised) float64 weights."""
    w = np.asarray(weights, dtype=np.float64)
    cdf = np.cumsum(w) / w.sum()
    # exact floor(cdf * 2^64) through (hi, lo) 32-bit halves (every step is exact in float64)
    x = cdf * 2.0 ** 32
    hi = np.floor(x)
    lo = np.floor((x - hi) * 2.0 ** 32)
    full = x >= 2.0 ** 32
    t = (np.where(full, 0, hi).astype(np.uint64) << np.uint64(32)) | np.where(full, 0, lo).astype(np.uint64)
    t[full] = np.uint64(M64)
    t[-1] = np.uint64(M64)
    return t


def draw(table: np.ndarray, u) -> np.ndarray:
    k = np.searchsorted(table, _u64(u), side="right")
    return np.minimum(k, len(table) - 1).astype(np.uint64)


@functools.lru_cache(maxsize=None)
def sm_table():
    """C2: 10% of the 148 SMs (SMs 0..14) take 50% of the records (Fig 2 imbalance)."""
    w = np.full(148, 0.5 / 133)
    w[:15] = 0.5 / 15
    return quantize_cdf(w)


@functools.lru_cache(maxsize=None)
def zipf_table(n: int, theta: float):
    k = np.arange(1, n + 1, dtype=np.float64)
    return quantize_cdf(k ** (-theta))


@functools.lru_cache(maxsize=None)
def tenant_table():
    return quantize_cdf([0.4, 0.3, 0.2, 0.1])


@functools.lru_cache(maxsize=None)
def c4_bounds():
    """bounds[4097]: bounds[0] = 2 MiB (end of the centroids); list sizes are heavy-tailed
    (Pareto alpha 1.2, >= 256 vectors) counts of 128-B vectors (uint8 SIFT, 128 dims), so list
    boundaries are not 512-B aligned and the 512-B warp records that cross them diverge."""
    u = rnd(LAYOUT_SEED, 20, np.arange(NLISTS)).astype(np.float64) / 2.0 ** 64
    vec = np.floor(256.0 / np.power(1.0 - u, 1.0 / 1.2))
    vec = np.clip(vec, 1, 1 << 22).astype(np.uint64)
    b = np.zeros(NLISTS + 1, dtype=np.uint64)
    b[0] = CENTROID_BYTES
    b[1:] = np.uint64(CENTROID_BYTES) + np.cumsum(vec * np.uint64(128))
    return b


def _common(seed, rec):
    return dict(block_id=(rnd(seed, 2, rec) % np.uint64(65536)),
                sm_id=(rnd(seed, 3, rec) % np.uint64(148)),
                warp_id=(rnd(seed, 4, rec) % np.uint64(64)))


def _fields_c1(seed, i, rec, lane, n_total):
    f = _common(seed, rec)
    f["addr"] = (rnd(seed, 1, i) & np.uint64(0xFFFFFFFF)) & ~np.uint64(7)
    f["size"] = np.full(i.shape, 8, dtype=np.uint64)
    f["kind"] = np.zeros(i.shape, dtype=np.uint64)
    return f


def _fields_c2(seed, i, rec, lane, n_total):
    sm = draw(sm_table(), rnd(seed, 3, rec))
    w = rnd(seed, 4, rec)
    warp = np.where(sm == 0, np.uint64(32) + w % np.uint64(32), w % np.uint64(64))
    base = (rnd(seed, 5, rec) & np.uint64(0xFFFFFFFFFF)) & ~np.uint64(0x1FF)
    return dict(block_id=rnd(seed, 2, rec) % np.uint64(65536), sm_id=sm, warp_id=warp,
                addr=base + np.uint64(16) * lane,
                size=np.uint64(1) << (rnd(seed, 7, rec) % np.uint64(5)),
                kind=np.zeros(i.shape, dtype=np.uint64))


def _fields_c3(seed, i, rec, lane, n_total):
    f = _common(seed, rec)
    prefill = np.uint64((n_total >> 5) // 4)
    is_pre = rec < prefill
    pre_page = rec % np.uint64(NWEIGHT)
    r2 = np.where(is_pre, np.uint64(0), rec - prefill)
    z = draw(zipf_table(NWEIGHT, 0.99), rnd(seed, 8, i))
    with np.errstate(over="ignore"):
        w_page = (z * np.uint64(PERM_A) + np.uint64(PERM_B)) % np.uint64(NWEIGHT)
    nkv = np.uint64(NPAGES - NWEIGHT)
    a = (r2 >> np.uint64(3)) % nkv
    back = rnd(seed, 9, i) % np.uint64(16)
    kv_page = np.uint64(NWEIGHT) + (a + nkv - back) % nkv
    is_w = (rnd(seed, 6, i) % np.uint64(5)) < np.uint64(4)
    dec_page = np.where(is_w, w_page, kv_page)
    off = rnd(seed, 1, i) & np.uint64(0xFF8)
    f["addr"] = np.where(is_pre, pre_page * np.uint64(4096) + lane * np.uint64(128),
                         dec_page * np.uint64(4096) + off)
    f["size"] = np.where(is_pre, np.uint64(128), np.uint64(8))
    f["kind"] = np.zeros(i.shape, dtype=np.uint64)
    return f


def _fields_c4(seed, i, rec, lane, n_total):
    f = _common(seed, rec)
    b = c4_bounds()
    data_bytes = b[NLISTS] - b[0]
    build = np.uint64((n_total >> 5) * 3 // 10)
    is_build = rec < build
    build_addr = b[0] + (rec * np.uint64(512)) % data_bytes + lane * np.uint64(16)
    q = np.where(is_build, np.uint64(0), rec - build)
    query, k = q // np.uint64(QUERY_RECS), q % np.uint64(QUERY_RECS)
    is_cent = k < np.uint64(64)
    cent_addr = (rnd(seed, 13, rec) % np.uint64(NLISTS)) * np.uint64(512) + lane * np.uint64(16)
    kk = np.where(is_cent, np.uint64(0), k - np.uint64(64))
    j, s = kk // np.uint64(32), kk % np.uint64(32)
    lst = draw(zipf_table(NLISTS, 0.8), rnd(seed, 12, query * np.uint64(16) + j))
    probe_addr = b[lst.astype(np.int64)] + s * np.uint64(512) + lane * np.uint64(16)
    probe_addr = np.minimum(probe_addr, b[NLISTS] - np.uint64(16))
    f["addr"] = np.where(is_build, build_addr, np.where(is_cent, cent_addr, probe_addr))
    f["size"] = np.full(i.shape, 16, dtype=np.uint64)
    f["kind"] = np.zeros(i.shape, dtype=np.uint64)
    return f


_FIELDS = {"C1": _fields_c1, "C2": _fields_c2, "C3": _fields_c3, "C4": _fields_c4}


def generate(config: str, seed: int, n: int, i0: int = 0, n_total: int | None = None) -> np.ndarray:
    """Events [i0, i0+n) of config `config` (global batch length n_total) as EVENT_DTYPE."""
    n_total = n if n_total is None else n_total
    i = np.arange(i0, i0 + n, dtype=np.uint64)
    rec, lane = i >> np.uint64(5), i & np.uint64(31)
    if config == "C5":
        tenant = draw(tenant_table(), rnd(seed, 10, rec))
        parts = [_FIELDS[c](seed, i, rec, lane, n_total) for c in ("C1", "C2", "C3", "C4")]
        f = {}
        for key in parts[0]:
            f[key] = np.choose(tenant.astype(np.int64), [p[key] for p in parts])
        is_fault = (tenant == np.uint64(2)) & (rnd(seed, 11, rec) % np.uint64(10) == np.uint64(0))
        f["kind"] = np.where(is_fault, np.uint64(2), np.uint64(0))
        f["size"] = np.where(is_fault, np.uint64(4096), f["size"])
        hook = f["kind"] | (tenant << np.uint64(8))
    else:
        f = _FIELDS[config](seed, i, rec, lane, n_total)
        hook = f["kind"]
    ev = np.zeros(n, dtype=EVENT_DTYPE)
    ev["addr"] = f["addr"]
    ev["ts"] = rec * np.uint64(1000)
    ev["hook"] = hook.astype(np.uint32)
    ev["block_id"] = f["block_id"].astype(np.uint32)
    ev["sm_id"] = f["sm_id"].astype(np.uint16)
    ev["warp_id"] = f["warp_id"].astype(np.uint8)
    ev["lane_id"] = lane.astype(np.uint8)
    ev["size"] = f["size"].astype(np.uint32)
    return ev


def records(n: int, **fields) -> np.ndarray:
    """Hand-built events: any EVENT_DTYPE field given as a scalar or array; lane_id defaults to i&31."""
    ev = np.zeros(n, dtype=EVENT_DTYPE)
    ev["lane_id"] = (np.arange(n) & 31).astype(np.uint8)
    for k, v in fields.items():
        ev[k] = v
    return ev


def c4_tables():
    """Host-written map contents for P4 (cfg[0], bounds[0..4096])."""
    return {"cfg": np.array([CENTROID_BYTES], dtype=np.uint64), "bounds": c4_bounds()}
