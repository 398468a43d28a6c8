"""Seeded synthetic workloads shaped like the paper's.

This module only draws random sequences, taxonomies and reads.  It holds none
of the method's arithmetic (no encoding, k-mers, hashing, sketching, tables,
ranking or classification) and is shared by the tests, bench.py and both
sides of the parity check (oracle/ and the CUDA path) as the single source of
inputs.  Every generator is a pure function of its seed.

Sequences are returned as ``(buf: uint8[total], offsets: uint64[n+1])`` —
the concatenated ASCII layout the C-ABI takes.

Taxonomy convention (mc.h): parent array, id 0 invalid, root = 1 with
parent[1] == 1.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import os

import numpy as np

ACGT = np.frombuffer(b"ACGT", dtype=np.uint8)
# complement lookup over all 256 byte values (non-ACGT -> 'N')
_COMP = np.full(256, ord("N"), dtype=np.uint8)
for a, b in zip(b"ACGTacgt", b"TGCAtgca"):
    _COMP[a] = b

REF_SEED = 21060815
READ_SEED = 81502106


@dataclass
class References:
    buf: np.ndarray            # uint8 ASCII, concatenated
    offsets: np.ndarray        # uint64 [n+1]
    target_ids: np.ndarray     # uint32 [n]
    taxa: np.ndarray           # uint32 [n]
    parent: np.ndarray         # uint32 [n_taxa]
    rank: np.ndarray           # uint8 [n_taxa] (0 root .. higher = lower rank)
    species_of_target: np.ndarray = field(default=None)

    @property
    def n(self) -> int:
        return int(self.target_ids.size)

    @property
    def total_bp(self) -> int:
        return int(self.offsets[-1])

    def seq(self, i: int) -> bytes:
        return self.buf[int(self.offsets[i]):int(self.offsets[i + 1])].tobytes()


@dataclass
class Reads:
    buf: np.ndarray
    offsets: np.ndarray
    mates_buf: np.ndarray | None = None
    mate_offsets: np.ndarray | None = None
    source_target: np.ndarray | None = None   # index into References (-1 = random)

    @property
    def n(self) -> int:
        return int(self.offsets.size - 1)

    @property
    def total_bp(self) -> int:
        t = int(self.offsets[-1])
        if self.mate_offsets is not None:
            t += int(self.mate_offsets[-1])
        return t


def random_bases(rng: np.random.Generator, n: int) -> np.ndarray:
    return ACGT[rng.integers(0, 4, size=n, dtype=np.uint8)]


def mutate(rng: np.random.Generator, seq: np.ndarray, rate: float) -> np.ndarray:
    """Copy of seq with ~rate substitutions (always to a different base)."""
    out = seq.copy()
    n_sub = rng.binomial(seq.size, rate) if rate > 0 else 0
    if n_sub:
        pos = rng.integers(0, seq.size, size=n_sub)
        cur = out[pos]
        code = np.searchsorted(ACGT, cur)  # ACGT is sorted: A<C<G<T
        code = np.where(ACGT[np.minimum(code, 3)] == cur, code, 0)
        out[pos] = ACGT[(code + rng.integers(1, 4, size=n_sub)) % 4]
    return out


def sprinkle_n(rng: np.random.Generator, seq: np.ndarray, rate: float, run: int = 1) -> None:
    n = rng.binomial(seq.size, rate) if rate > 0 else 0
    if n:
        pos = rng.integers(0, seq.size, size=n)
        for r in range(run):
            seq[np.minimum(pos + r, seq.size - 1)] = ord("N")


def revcomp(a: np.ndarray) -> np.ndarray:
    return _COMP[a[::-1]]


def concat(seqs) -> tuple[np.ndarray, np.ndarray]:
    offs = np.zeros(len(seqs) + 1, np.uint64)
    offs[1:] = np.cumsum([s.size for s in seqs], dtype=np.uint64)
    buf = np.empty(int(offs[-1]), np.uint8)
    for i, s in enumerate(seqs):
        buf[int(offs[i]):int(offs[i + 1])] = s
    return buf, offs


# --------------------------------------------------------------------------
# taxonomies
# --------------------------------------------------------------------------
class TaxBuilder:
    def __init__(self):
        self.parent = [0, 1]   # 0 invalid, 1 = root
        self.rank = [255, 0]

    def add(self, parent: int, rank: int) -> int:
        self.parent.append(parent)
        self.rank.append(rank)
        return len(self.parent) - 1

    def arrays(self):
        return np.asarray(self.parent, np.uint32), np.asarray(self.rank, np.uint8)


# --------------------------------------------------------------------------
# configs[0] "tiny": 8 genomes x 200 kbp, 3-level taxonomy
# --------------------------------------------------------------------------
def tiny_references(seed: int = REF_SEED, n_genomes: int = 8, length: int = 200_000) -> References:
    rng = np.random.default_rng(seed)
    tb = TaxBuilder()
    fams = [tb.add(1, 1) for _ in range(2)]
    gens = [tb.add(fams[i // 2], 2) for i in range(4)]
    species = [tb.add(gens[i * 4 // n_genomes], 3) for i in range(n_genomes)]
    seqs = [random_bases(rng, length) for _ in range(n_genomes)]
    buf, offs = concat(seqs)
    parent, rank = tb.arrays()
    return References(buf, offs, np.arange(n_genomes, dtype=np.uint32), np.asarray(species, np.uint32),
                      parent, rank, np.arange(n_genomes))


# --------------------------------------------------------------------------
# strain-structured references ("small" / configs[1] "bacterial subset")
#   genus ancestor -> species (species_div subs) -> strains (0.5-1% subs)
#   strains per species ~ Zipf(zipf_a) capped; optional plasmids; rare N runs
# --------------------------------------------------------------------------
def strain_references(seed=REF_SEED, n_targets: int = 1000, median_len: float = 4e6,
                      min_len: int = 1_000_000, max_len: int = 10_000_000, n_genera: int | None = None,
                      species_div: float = 0.10, strain_div=(0.005, 0.01), zipf_a: float = 1.2,
                      max_strains: int = 64, plasmid_frac: float = 0.05, n_rate: float = 1e-5,
                      id_stride: int = 1, id_offset: int = 0, tb: TaxBuilder | None = None,
                      sequences: bool = True) -> References:
    """Strain-structured references.  With a shared ``tb`` several shards can
    extend one taxonomy; ``sequences=False`` builds only the taxonomy part
    (same random structure, no bases) so every rank can reproduce the global
    taxonomy without generating the other shards' genomes."""
    srng = np.random.default_rng(seed if not isinstance(seed, tuple) else list(seed))
    rng = np.random.default_rng([*(seed if isinstance(seed, tuple) else (seed,)), 7])
    tb = TaxBuilder() if tb is None else tb
    strains = []
    n_chrom = int(round(n_targets * (1 - plasmid_frac)))
    while sum(strains) < n_chrom:
        strains.append(int(min(max_strains, srng.zipf(zipf_a))))
    strains[-1] -= sum(strains) - n_chrom
    n_species = len(strains)
    if n_genera is None:
        n_genera = max(1, n_species // 4)
    n_fam = max(1, n_genera // 4)
    fams = [tb.add(1, 1) for _ in range(n_fam)]
    gens = [tb.add(fams[g % n_fam], 2) for g in range(n_genera)]
    genus_of_species = srng.integers(0, n_genera, size=n_species)
    sp_tax = [tb.add(gens[genus_of_species[s]], 3) for s in range(n_species)]
    glen = np.clip(srng.lognormal(np.log(median_len), 0.5, size=n_genera), min_len, max_len).astype(np.int64)
    taxa, species_of, lens = [], [], []
    for s in range(n_species):
        for _ in range(strains[s]):
            taxa.append(tb.add(sp_tax[s], 4))
            species_of.append(s)
            lens.append(int(glen[genus_of_species[s]]))
    for _ in range(n_targets - len(taxa)):  # plasmids: short unique targets of random species
        s = int(srng.integers(0, n_species))
        taxa.append(tb.add(sp_tax[s], 4))
        species_of.append(s)
        lens.append(int(srng.integers(5_000, 200_000)))
    order = srng.permutation(len(taxa))  # insertion order interleaves species (like RefSeq files)
    ids = (np.arange(len(taxa), dtype=np.uint64) * id_stride + id_offset).astype(np.uint32)
    parent, rank = tb.arrays()
    if not sequences:
        offs = np.zeros(len(taxa) + 1, np.uint64)
        offs[1:] = np.cumsum(np.asarray(lens, np.uint64)[order])
        return References(np.zeros(0, np.uint8), offs, ids, np.asarray(taxa, np.uint32)[order], parent, rank,
                          np.asarray(species_of)[order])
    seqs = [None] * len(taxa)
    genus_seq, i = {}, 0
    for s in range(n_species):
        g = int(genus_of_species[s])
        if g not in genus_seq:
            genus_seq[g] = random_bases(rng, int(glen[g]))
        sp = mutate(rng, genus_seq[g], species_div)
        for _ in range(strains[s]):
            st = mutate(rng, sp, rng.uniform(*strain_div))
            sprinkle_n(rng, st, n_rate, run=int(rng.integers(1, 20)))
            seqs[i] = st
            i += 1
        del sp
    for j in range(i, len(taxa)):
        seqs[j] = random_bases(rng, lens[j])
    seqs = [seqs[j] for j in order]
    buf, offs = concat(seqs)
    return References(buf, offs, ids, np.asarray(taxa, np.uint32)[order], parent, rank,
                      np.asarray(species_of)[order])


def scaffold_references(seed=REF_SEED + 31, n_species: int = 8, chrom_len: int = 3_000_000,
                        scaffolds_per_species: int = 2500, scaffold_median: float = 2000,
                        n_rate: float = 2e-4) -> References:
    """AFS31-shaped eukaryotic references (SURVEY.md §8(f) NEXT rank 4, P:800-805,
    T1 P:764-765): per species one long chromosome plus thousands of short
    scaffold targets (log-normal lengths, many shorter than one window) with
    N runs; insertion order interleaves species.  Stresses target counts,
    ranked-window ids and tiny targets many to a warp."""
    rng = np.random.default_rng((seed, 31))
    tb = TaxBuilder()
    fam = tb.add(1, 1)
    gen = [tb.add(fam, 2) for _ in range(max(1, n_species // 3))]
    taxa, species_of, seqs = [], [], []
    for s in range(n_species):
        sp = tb.add(gen[s % len(gen)], 3)
        chrom = random_bases(rng, chrom_len)
        sprinkle_n(rng, chrom, n_rate, run=int(rng.integers(1, 200)))
        taxa.append(tb.add(sp, 4))
        species_of.append(s)
        seqs.append(chrom)
        lens = np.clip(rng.lognormal(np.log(scaffold_median), 1.0, size=scaffolds_per_species), 20, 60_000)
        for L in lens.astype(np.int64):
            sc = random_bases(rng, int(L))
            sprinkle_n(rng, sc, n_rate, run=int(rng.integers(1, 50)))
            taxa.append(tb.add(sp, 4))
            species_of.append(s)
            seqs.append(sc)
    order = rng.permutation(len(seqs))
    seqs = [seqs[j] for j in order]
    buf, offs = concat(seqs)
    parent, rank = tb.arrays()
    ids = (np.arange(len(seqs), dtype=np.uint64) * 3 + 11).astype(np.uint32)
    return References(buf, offs, ids, np.asarray(taxa, np.uint32)[order], parent, rank,
                      np.asarray(species_of)[order])


def afs31_shard(shard: int = 0, n_shards: int = 8, seed: int = REF_SEED, scale: float = 1.0) -> References:
    """All-Food-Seq-31-shaped eukaryotic database (Table 1: 31 species,
    77 GB; animal and plant genomes of much longer sequences, some
    only at scaffold level -> hundreds of thousands of targets per genome),
    cut into n_shards target shards (species s -> shard s mod n_shards).
      * genome sizes log-uniform in [0.4, 6] Gbp, rescaled to 77 Gbp in all
        (x scale);
      * every third species (s mod 3 == 0) is scaffold-level: its genome is
        cut into scaffolds of log-normal length (median 4 kbp, sigma 1.6,
        clipped to [200 bp, 2 Mbp]) -> ~10^5 targets per genome; the others
        are chromosome-level (8-40 chromosomes, Dirichlet proportions);
      * N runs at rate 1e-4 (assembly gaps).
    All sequences of a genome share the genome's taxon (rank 4, under its
    species -> genus -> family -> root).  Every rank rebuilds the global
    taxonomy from the seeded structure; only the shard's bases are generated,
    each species from its own counter-seeded stream.  Target ids: shard * 2^24 + i."""
    srng = np.random.default_rng((seed, 31))
    n_sp = 31
    g = np.exp(srng.uniform(np.log(0.4e9), np.log(6e9), size=n_sp))
    g = np.maximum((g * (77e9 * scale / g.sum())).astype(np.int64), 20_000)
    n_chr = srng.integers(8, 41, size=n_sp)
    tb = TaxBuilder()
    fams = [tb.add(1, 1) for _ in range(4)]
    genome_tax = []
    for s in range(n_sp):
        genus = tb.add(fams[s % 4], 2)
        genome_tax.append(tb.add(tb.add(genus, 3), 4))
    seqs_len, taxa, species_of, parts = [], [], [], []
    for s in range(shard, n_sp, n_shards):
        rng = np.random.default_rng((seed, 31, s))
        genome = random_bases(rng, int(g[s]))
        sprinkle_n(rng, genome, 1e-4, run=int(rng.integers(10, 200)))
        if s % 3 == 0:
            lens = []
            left = int(g[s])
            while left > 0:
                x = np.clip(rng.lognormal(np.log(4000), 1.6, size=4096), 200, 2e6).astype(np.int64)
                c = np.cumsum(x)
                k = int(np.searchsorted(c, left))
                lens.append(x[:k + 1])
                left -= int(c[min(k, c.size - 1)])
            lens = np.concatenate(lens)
            lens[-1] -= int(lens.sum()) - int(g[s])
            lens = lens[lens > 0]
        else:
            lens = np.maximum(rng.dirichlet(np.full(int(n_chr[s]), 2.0)) * g[s], 1).astype(np.int64)
            lens[-1] += int(g[s]) - int(lens.sum())
        parts.append(genome)
        seqs_len.append(lens)
        taxa.append(np.full(lens.size, genome_tax[s], np.uint32))
        species_of.append(np.full(lens.size, s, np.int64))
    lens = np.concatenate(seqs_len)
    offs = np.zeros(lens.size + 1, np.uint64)
    offs[1:] = np.cumsum(lens, dtype=np.uint64)
    buf = np.concatenate(parts) if len(parts) > 1 else parts[0]
    parent, rank = tb.arrays()
    ids = (np.uint32(shard) << np.uint32(24)) + np.arange(lens.size, dtype=np.uint32)
    return References(buf, offs, ids, np.concatenate(taxa), parent, rank, np.concatenate(species_of))


def refseq_shard(shard: int = 0, n_shards: int = 8, seed: int = REF_SEED, scale: float = 1.0) -> References:
    """configs[3] "RefSeq Release 202-shaped" (Table 1; SURVEY
    §8(d)): ~51k sequences of ~15.5k species, ~74 Gbp in all, cut into
    n_shards target shards (one per GPU; shard = genus mod n_shards, so a
    genus -- and every strain of its species -- lives in one shard).
      * ~9,000 viral species: one 10-200 kbp genome each (log-uniform);
      * ~6,360 bacterial/archaeal species in 1,600 genera: genus ancestor
        (log-normal, median 3.3 Mbp, 2-13 Mbp) -> species (10 % subs) ->
        strains (0.5-1 % subs, N runs), strains per species ~ Zipf(2.1) capped
        at 100 (~20k genomes); each genome also carries Poisson(1) plasmids (5-200 kbp);
      * 100 fungal species: 8-16 chromosomes totalling 10-40 Mbp.
    Taxonomy: target -> species -> genus -> family -> root (every rank
    rebuilds the global one from the seeded structure; only the shard's bases
    are generated).  ``scale`` shrinks the species counts (tests)."""
    srng = np.random.default_rng((seed, 202))
    tb = TaxBuilder()
    n_vir, n_bac, n_fun = (max(1, int(round(x * scale))) for x in (9000, 6360, 100))
    g_vir, g_bac, g_fun = (max(1, int(round(x * scale))) for x in (900, 1600, 40))
    fam = {k: [tb.add(1, 1) for _ in range(max(1, g // 8))] for k, g in (("v", g_vir), ("b", g_bac), ("f", g_fun))}
    genera = []  # (kind, genus taxon, global genus index)
    for k, g in (("v", g_vir), ("b", g_bac), ("f", g_fun)):
        for i in range(g):
            genera.append((k, tb.add(fam[k][i % len(fam[k])], 2), len(genera)))
    by_kind = {k: [x for x in genera if x[0] == k] for k in "vbf"}
    targets = []  # (taxon, length, genus index, species index, role, seed tag)
    n_sp = 0
    for k, n in (("v", n_vir), ("b", n_bac), ("f", n_fun)):
        gs = by_kind[k]
        for j in range(n):
            gk, gtax, gi = gs[int(srng.integers(0, len(gs)))] if j >= len(gs) else gs[j]
            sp = tb.add(gtax, 3)
            if k == "v":
                L = int(np.exp(srng.uniform(np.log(10_000), np.log(200_000))))
                targets.append((tb.add(sp, 4), L, gi, n_sp, "v", len(targets)))
            elif k == "b":
                for _ in range(int(min(100, srng.zipf(2.1)))):
                    targets.append((tb.add(sp, 4), 0, gi, n_sp, "c", len(targets)))  # chromosome: genus length
                    for _ in range(int(srng.poisson(1.0))):
                        L = int(np.exp(srng.uniform(np.log(5_000), np.log(200_000))))
                        targets.append((tb.add(sp, 4), L, gi, n_sp, "p", len(targets)))
            else:
                nc = int(srng.integers(8, 17))
                tot = srng.uniform(10e6, 40e6)
                for L in srng.dirichlet(np.ones(nc) * 4) * tot:
                    targets.append((tb.add(sp, 4), int(L), gi, n_sp, "f", len(targets)))
            n_sp += 1
    glen = np.clip(srng.lognormal(np.log(3.3e6), 0.4, size=len(genera)), 2e6, 13e6).astype(np.int64)
    order = srng.permutation(len(targets))  # insertion order interleaves species (like RefSeq files)
    mine = [int(i) for i in order if targets[int(i)][2] % n_shards == shard]
    parent, rank = tb.arrays()
    seqs, anc, spseq = [], {}, {}
    # bases: per-genus / per-species / per-target seeded generators, so a shard
    # reproduces exactly the sequences it owns
    for i in mine:
        tax, L, gi, si, role, tag = targets[i]
        trng = np.random.default_rng((seed, 202, 3, tag))
        if role == "c":
            if si not in spseq:
                if gi not in anc:
                    anc[gi] = random_bases(np.random.default_rng((seed, 202, 1, gi)), int(glen[gi]))
                spseq[si] = mutate(np.random.default_rng((seed, 202, 2, si)), anc[gi], 0.10)
            st = mutate(trng, spseq[si], trng.uniform(0.005, 0.01))
            sprinkle_n(trng, st, 1e-5, run=int(trng.integers(1, 20)))
            seqs.append(st)
        else:
            seqs.append(random_bases(trng, L))
    buf, offs = concat(seqs)
    ids = np.asarray(mine, np.uint32)  # global target index: unique across shards
    taxa = np.asarray([targets[i][0] for i in mine], np.uint32)
    species_of = np.asarray([targets[i][3] for i in mine], np.int64)
    return References(buf, offs, ids, taxa, parent, rank, species_of)


def subset_shard(shard: int = 0, n_shards: int = 1, seed: int = REF_SEED, n_targets: int = 1000,
                 **kw) -> References:
    """configs[1] "bacterial subset" (~1,000 genomes, ~4 Gbp) -- one shard per
    rank for the weak-scaling multi-GPU run.  Shards share one global taxonomy
    (every rank rebuilds all shards' taxonomy parts, cheap) and use disjoint
    target ids (shard * 2^24 + i).  Strain counts ~ Zipf(2.0) capped at 300,
    so a few species have 100+ strains and their features exceed the cap."""
    kw.setdefault("zipf_a", 2.0)
    kw.setdefault("max_strains", 300)
    tb = TaxBuilder()
    mine = None
    for s in range(n_shards):
        r = strain_references(seed=(seed, s), n_targets=n_targets, tb=tb, sequences=(s == shard),
                              id_offset=s << 24, **kw)
        if s == shard:
            mine = r
    mine.parent, mine.rank = tb.arrays()
    return mine


# --------------------------------------------------------------------------
# reads
# --------------------------------------------------------------------------
def _cut(rng, refs: References, n: int, frag_len: np.ndarray, weights: np.ndarray | None = None):
    lens = np.diff(refs.offsets).astype(np.int64)
    ok = lens >= frag_len.max()
    w = np.where(ok, lens if weights is None else weights, 0).astype(np.float64)
    tgt = rng.choice(refs.n, size=n, p=w / w.sum())
    start = refs.offsets[tgt].astype(np.int64) + (rng.random(n) * (lens[tgt] - frag_len + 1)).astype(np.int64)
    return tgt, start


def _errors(rng, a: np.ndarray, sub_rate: float, n_rate: float) -> None:
    if sub_rate > 0:
        m = rng.random(a.shape) < sub_rate
        if m.any():
            cur = a[m]
            code = np.searchsorted(ACGT, cur)
            code = np.minimum(code, 3)
            a[m] = ACGT[(code + rng.integers(1, 4, size=cur.size)) % 4]
    if n_rate > 0:
        m = rng.random(a.shape) < n_rate
        a[m] = ord("N")


def single_end_reads(refs: References, n: int, length: int = 100, seed: int = READ_SEED,
                     random_frac: float = 0.10, sub_rate: float = 0.005, n_rate: float = 0.0005,
                     length_range: tuple[int, int] | None = None) -> Reads:
    """configs[0]: 90% cut from the references (uniform position, random
    strand, substitutions, Ns), 10% random (unclassifiable).  With
    length_range, lengths are uniform in [lo, hi] (HiSeq/MiSeq-like)."""
    rng = np.random.default_rng(seed)
    if length_range is None:
        lens = np.full(n, length, np.int64)
    else:
        lens = rng.integers(length_range[0], length_range[1] + 1, size=n)
    maxlen = int(lens.max()) if n else 0
    is_rand = rng.random(n) < random_frac
    tgt, start = _cut(rng, refs, n, np.full(n, maxlen, np.int64))
    idx = start[:, None] + np.arange(maxlen)[None, :]
    mat = refs.buf[idx]
    rev = rng.random(n) < 0.5
    mat[rev] = _COMP[mat[rev][:, ::-1]]
    if is_rand.any():
        mat[is_rand] = ACGT[rng.integers(0, 4, size=(int(is_rand.sum()), maxlen), dtype=np.uint8)]
    _errors(rng, mat, sub_rate, n_rate)
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum(lens, dtype=np.uint64)
    keep = np.arange(maxlen)[None, :] < lens[:, None]
    buf = mat[keep]
    src = np.where(is_rand, -1, tgt)
    return Reads(buf, offs, source_target=src)


def paired_reads(refs: References, n: int, length: int = 150, insert_mean: float = 400, insert_sd: float = 50,
                 seed: int = READ_SEED, sub_rate: float = 0.005, n_rate: float = 0.0, random_frac: float = 0.0,
                 chunk: int = 200_000, target_weights: np.ndarray | None = None) -> Reads:
    """configs[1]: pairs 2 x length, insert ~ N(mean, sd), mate 2 reverse-
    complemented, substitutions.  Generated in chunks to bound host memory.
    target_weights: per-target sampling weights (default: target length)."""
    rng = np.random.default_rng(seed)
    b1 = np.empty(n * length, np.uint8)
    b2 = np.empty(n * length, np.uint8)
    src = np.empty(n, np.int64)
    for c0 in range(0, n, chunk):
        c = min(chunk, n - c0)
        ins = np.clip(rng.normal(insert_mean, insert_sd, size=c), length, None).astype(np.int64)
        tgt, start = _cut(rng, refs, c, ins, target_weights)
        a = start[:, None] + np.arange(length)[None, :]
        m1 = refs.buf[a]
        e = (start + ins - length)[:, None] + np.arange(length)[None, :]
        m2 = refs.buf[e]
        m2 = _COMP[m2[:, ::-1]]
        flip = rng.random(c) < 0.5           # fragment from the reverse strand
        t = m1[flip].copy()
        m1[flip] = m2[flip]
        m2[flip] = t
        is_rand = rng.random(c) < random_frac
        if is_rand.any():
            k = int(is_rand.sum())
            m1[is_rand] = ACGT[rng.integers(0, 4, size=(k, length), dtype=np.uint8)]
            m2[is_rand] = ACGT[rng.integers(0, 4, size=(k, length), dtype=np.uint8)]
        _errors(rng, m1, sub_rate, n_rate)
        _errors(rng, m2, sub_rate, n_rate)
        b1[c0 * length:(c0 + c) * length] = m1.reshape(-1)
        b2[c0 * length:(c0 + c) * length] = m2.reshape(-1)
        src[c0:c0 + c] = np.where(is_rand, -1, tgt)
    offs = np.arange(n + 1, dtype=np.uint64) * np.uint64(length)
    return Reads(b1, offs, b2, offs.copy(), src)


def afs_reads(refs: References, n: int, n_species: int = 20, length: int = 101, seed: int = READ_SEED + 20,
              **kw) -> Reads:
    """configs[2] "AFS20-shaped" mock community: pairs from n_species species
    of the database with log-normal abundances (sigma 1); within a species,
    targets (strains) are drawn proportionally to their length.  2 x 101 bp
    (the read length is not given for AFS; SURVEY.md §8(d) proposal)."""
    rng = np.random.default_rng((seed, 20))
    sp = np.unique(refs.species_of_target)
    pick = rng.choice(sp, size=min(n_species, sp.size), replace=False)
    ab = dict(zip(pick.tolist(), rng.lognormal(0.0, 1.0, size=pick.size).tolist()))
    lens = np.diff(refs.offsets).astype(np.float64)
    w = np.zeros(refs.n)
    for s_ in pick.tolist():
        m = refs.species_of_target == s_
        w[m] = ab[s_] * lens[m] / lens[m].sum()
    return paired_reads(refs, n, length=length, insert_mean=300, insert_sd=40, seed=seed, target_weights=w, **kw)


def kal_reads(refs: References, n: int, length: int = 101, seed: int = READ_SEED + 30, absent_frac: float = 0.95,
              **kw) -> Reads:
    """configs[4] "KAL_D-shaped": 2 x 101 bp pairs, ~95 % from genomes absent
    from the database (few hits; random sequence here) and 5 % cut
    from database targets."""
    return paired_reads(refs, n, length=length, insert_mean=300, insert_sd=40, seed=seed, random_frac=absent_frac,
                        **kw)


_FORK = {}  # references + shared output buffers, inherited (not pickled) by forked workers


def _kal_chunk(args):
    n, length, seed, i, chunk = args
    r = kal_reads(_FORK["refs"], n, length=length, seed=(seed, i))
    lo = i * chunk * length
    _FORK["b1"][lo:lo + r.buf.size] = r.buf
    _FORK["b2"][lo:lo + r.mates_buf.size] = r.mates_buf
    return i


def kal_stream(refs: References, n: int, length: int = 101, seed: int = READ_SEED + 60, chunk: int = 1_000_000,
               workers: int | None = None) -> Reads:
    """configs[4] at its stated size: n (>= 50M) KAL_D-shaped pairs, generated
    in chunks of `chunk` pairs (chunk i seeded (seed, i), so the stream is the
    same whatever the worker count) by forked host workers writing into shared
    memory."""
    import concurrent.futures as cf
    import mmap
    import multiprocessing as mp
    nch = (n + chunk - 1) // chunk
    m1, m2 = mmap.mmap(-1, max(n * length, 1)), mmap.mmap(-1, max(n * length, 1))  # MAP_SHARED | MAP_ANONYMOUS
    _FORK.update(refs=refs, b1=np.frombuffer(m1, np.uint8), b2=np.frombuffer(m2, np.uint8))
    jobs = [(min(chunk, n - i * chunk), length, seed, i, chunk) for i in range(nch)]
    workers = workers or max(1, min(nch, len(os.sched_getaffinity(0))))
    try:
        if workers == 1:
            for j in jobs:
                _kal_chunk(j)
        else:
            with cf.ProcessPoolExecutor(workers, mp_context=mp.get_context("fork")) as ex:
                list(ex.map(_kal_chunk, jobs))
        b1, b2 = _FORK["b1"], _FORK["b2"]  # (views keep the shared mappings alive)
    finally:
        _FORK.clear()
    offs = np.arange(n + 1, dtype=np.uint64) * np.uint64(length)
    return Reads(b1, offs, b2, offs.copy())


def variable_reads(refs: References, n: int, min_len: int, max_len: int, mean_len: float,
                   seed: int = READ_SEED + 40, sub_rate: float = 0.005, chunk: int = 200_000) -> Reads:
    """Single-end reads of variable length shaped like the paper's HiSeq
    (19-101 bp, mean 92.3) and MiSeq (19-251 bp, mean 156.8) sets (Table 2,
    P:766-769): a length is max_len with probability p, else uniform in
    [min_len, max_len], p chosen so the mean is mean_len.  Cut from the
    references (uniform position, random strand) with substitutions; chunked."""
    rng = np.random.default_rng((seed, min_len, max_len))
    mid = (min_len + max_len) / 2.0
    p = min(1.0, max(0.0, (mean_len - mid) / (max_len - mid)))
    lens = np.where(rng.random(n) < p, max_len, rng.integers(min_len, max_len + 1, size=n)).astype(np.int64)
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum(lens, dtype=np.uint64)
    buf = np.empty(int(offs[-1]), np.uint8)
    src = np.empty(n, np.int64)
    for c0 in range(0, n, chunk):
        c = min(chunk, n - c0)
        tgt, start = _cut(rng, refs, c, np.full(c, max_len, np.int64))
        mat = refs.buf[start[:, None] + np.arange(max_len)[None, :]]
        rev = rng.random(c) < 0.5
        mat[rev] = _COMP[mat[rev][:, ::-1]]
        _errors(rng, mat, sub_rate, 0.0)
        keep = np.arange(max_len)[None, :] < lens[c0:c0 + c, None]
        buf[int(offs[c0]):int(offs[c0 + c])] = mat[keep]
        src[c0:c0 + c] = tgt
    return Reads(buf, offs, source_target=src)


def hiseq_reads(refs: References, n: int, seed: int = READ_SEED + 40, **kw) -> Reads:
    """HiSeq-shaped: single-end 19-101 bp, mean 92.3 (Table 2)."""
    return variable_reads(refs, n, 19, 101, 92.3, seed=seed, **kw)


def miseq_reads(refs: References, n: int, seed: int = READ_SEED + 50, **kw) -> Reads:
    """MiSeq-shaped: single-end 19-251 bp, mean 156.8 (Table 2)."""
    return variable_reads(refs, n, 19, 251, 156.8, seed=seed, **kw)


def reads_from_list(r1, r2=None) -> Reads:
    def cat(lst):
        arrs = [np.frombuffer(s.encode() if isinstance(s, str) else bytes(s), np.uint8) for s in lst]
        return concat(arrs) if arrs else (np.zeros(0, np.uint8), np.zeros(1, np.uint64))
    b1, o1 = cat(r1)
    if r2 is None:
        return Reads(b1, o1)
    b2, o2 = cat(r2)
    return Reads(b1, o1, b2, o2)


def references_from_list(seqs, taxa, parent, ids=None) -> References:
    arrs = [np.frombuffer(s.encode() if isinstance(s, str) else bytes(s), np.uint8) for s in seqs]
    buf, offs = concat(arrs)
    n = len(seqs)
    ids = np.arange(n, dtype=np.uint32) if ids is None else np.asarray(ids, np.uint32)
    parent = np.asarray(parent, np.uint32)
    return References(buf, offs, ids, np.asarray(taxa, np.uint32), parent, np.zeros(parent.size, np.uint8))
