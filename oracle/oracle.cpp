// ============================================================================
// MetaCache oracle — plain, slow, obviously-correct CPU implementation.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// The product path (paper_2106_08150_b200/) never links, imports or calls it,
// and it shares no code, header, table or constant generator with the CUDA
// path.  It is single-threaded, except two variants that only split
// independent work over host threads: the feature-restricted full-size build
// (sketches targets in parallel, appends in insertion order) and the query
// over contiguous record slices (or_classify_threads, the N-thread timing of
// bench.py's cpu_baseline; same results as or_classify).  It uses std::map / std::vector / std::set and
// follows the paper's steps in the paper's order (arXiv 2106.08150,
// /root/reference/PAPER.md, cited as P:<line>).
//
// Readings of silent / garbled points are those of SURVEY.md §8(c) (S1..S24),
// restated in DESIGN.md "Readings".
//
// Pins (tests/test_oracle_*.py, -m "not gpu"):
//   encode/canonical : brute force vs Python string reverse-complement,
//                      canon(x) == canon(rc(x)) over all 4^4 4-mers
//   windows          : closed form ceil((L-k+1)/stride), exact cover
//   sketch           : paper toy example P:191-197 (tests/golden/minhash_toy.json),
//                      brute force with a random lookup-table hash
//   h1               : bijectivity (inverse mixer) -- VALUES parity unpinned
//                      (the hash is a choice, S1)
//   table + cap      : brute-force multiset, "254 smallest" rule
//   top hits + merge : Figure 1 worked example P:336-435
//                      (tests/golden/fig1_candidates.json), brute-force ranges
//   classify / LCA   : hand-made trees, exact self-classification
//   sws (S10 / S25)  : closed form with window-aligned mates, paired and
//                      single-end, with and without insert_size_max
//   partition plan   : S9 incl. explicitly placed targets' bp
// ============================================================================
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <thread>
#include <vector>

namespace {

// ---- §5.2 step (1), P:681-682 and §5.3: nucleotide encoding ------
// S3/S4: A=0 C=1 G=2 T=3 (case-insensitive); any other char is ambiguous (-1).
int base_code(char c) {
    switch (c) {
        case 'A': case 'a': return 0;
        case 'C': case 'c': return 1;
        case 'G': case 'g': return 2;
        case 'T': case 't': return 3;
        default: return -1;
    }
}

char complement(char c) {
    switch (c) {
        case 'A': case 'a': return 'T';
        case 'C': case 'c': return 'G';
        case 'G': case 'g': return 'C';
        case 'T': case 't': return 'A';
        default: return 'N';
    }
}

// k-mer value with the first base most significant (S3): sum c_j * 4^(k-1-j).
// Returns false if the k-mer holds an ambiguous base (S4: skipped).
bool encode_kmer(const std::string& kmer, uint32_t* out) {
    uint64_t v = 0;
    for (char c : kmer) {
        int b = base_code(c);
        if (b < 0) return false;
        v = v * 4 + (uint64_t)b;
    }
    *out = (uint32_t)v;
    return true;
}

std::string reverse_complement(const std::string& s) {
    std::string r(s.rbegin(), s.rend());
    for (char& c : r) c = complement(c);
    return r;
}

}  // namespace

extern "C" {

// ---- S1: h1 -- the paper never defines it; our reading is a
// 32-bit bijective integer mixer.  VALUES are parity-unpinned (a choice).
uint32_t or_h1(uint32_t x) {
    x = ((x >> 16) ^ x) * 0x45d9f3bu;
    x = ((x >> 16) ^ x) * 0x45d9f3bu;
    x = (x >> 16) ^ x;
    return x;
}

// ---- §4.1, §5.2: windows ---------------------------
// n = L-k+1 k-mer starts; window j holds starts [j*stride, min((j+1)*stride, n)).
uint64_t or_window_count(uint64_t L, uint32_t k, uint32_t w) {
    if (L < k) return 0;
    uint64_t n = L - k + 1, stride = w - k + 1;
    return (n + stride - 1) / stride;
}

// canonical value of a k-mer given as a string: min(fwd, rc).
// Returns 0 and sets *ok=0 if ambiguous.
uint32_t or_canonical_kmer(const char* kmer, uint32_t k, int* ok) {
    std::string s(kmer, kmer + k);
    uint32_t f = 0, r = 0;
    if (!encode_kmer(s, &f) || !encode_kmer(reverse_complement(s), &r)) {
        *ok = 0;
        return 0;
    }
    *ok = 1;
    return std::min(f, r);
}

// Sketch parameters.  `table` (optional, 4^k entries) replaces h1 by a lookup
// so that the paper's toy example P:191-197 (which prints its own hash values
// and does not canonicalise) can be reproduced; `canonical`=0 disables the
// canonical step for that example only.
struct or_sketch_params {
    uint32_t k, s, w;
    uint32_t canonical;
    const uint32_t* table;
};

}  // extern "C"

namespace {

// ---- §4.1 P:330-333 + §5.2 steps (1)-(3) + S6: sketch of one window --------
// All valid k-mers of the window -> canonical -> h1 -> sorted unique -> first s.
std::vector<uint32_t> sketch_window(const or_sketch_params& p, const std::string& seq,
                                    uint64_t first_start, uint64_t end_start) {
    std::set<uint32_t> feats;  // ordered, unique
    for (uint64_t i = first_start; i < end_start; ++i) {
        std::string km = seq.substr(i, p.k);
        uint32_t fwd = 0;
        if (!encode_kmer(km, &fwd)) continue;  // S4: skip ambiguous k-mers
        uint32_t val = fwd;
        if (p.canonical) {
            uint32_t rc = 0;
            encode_kmer(reverse_complement(km), &rc);
            val = std::min(fwd, rc);
        }
        feats.insert(p.table ? p.table[val] : or_h1(val));
    }
    std::vector<uint32_t> out;
    for (uint32_t f : feats) {
        if (out.size() == p.s) break;
        out.push_back(f);
    }
    return out;
}

std::vector<std::vector<uint32_t>> sketch_sequence(const or_sketch_params& p, const std::string& seq) {
    std::vector<std::vector<uint32_t>> res;
    uint64_t L = seq.size();
    uint64_t nwin = or_window_count(L, p.k, p.w);
    uint64_t n = L >= p.k ? L - p.k + 1 : 0, stride = p.w - p.k + 1;
    for (uint64_t j = 0; j < nwin; ++j) {
        uint64_t b = j * stride, e = std::min((j + 1) * stride, n);
        res.push_back(sketch_window(p, seq, b, e));
    }
    return res;
}

}  // namespace

extern "C" {

// Sketch every window of one sequence.  out_feats: nwin*s (rows padded with 0),
// out_counts: nwin.  Returns nwin.
uint64_t or_sketch_sequence(const or_sketch_params* p, const char* seq, uint64_t len,
                            uint32_t* out_feats, uint32_t* out_counts) {
    std::string s(seq, seq + len);
    auto sk = sketch_sequence(*p, s);
    for (size_t j = 0; j < sk.size(); ++j) {
        if (out_counts) out_counts[j] = (uint32_t)sk[j].size();
        if (out_feats)
            for (uint32_t i = 0; i < p->s; ++i)
                out_feats[j * p->s + i] = i < sk[j].size() ? sk[j][i] : 0u;
    }
    return sk.size();
}

// ---- S9: deterministic partition assignment (P:444-452 reading) ------------
// Greedy by bp in insertion order: each target goes to the partition holding
// the fewest bp so far, ties to the lowest index.  running_bp (P entries) is
// in/out so that successive insert batches continue the same greedy run.
void or_plan_partitions(uint32_t P, uint32_t n, const uint64_t* lengths, uint64_t* running_bp,
                        uint32_t* out_part) {
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t best = 0;
        for (uint32_t q = 1; q < P; ++q)
            if (running_bp[q] < running_bp[best]) best = q;
        out_part[i] = best;
        running_bp[best] += lengths[i];
    }
}

// ---- D8 candidate: (target, hits, [win_beg, win_end]) Fig. 1 P:389-394 -----
struct or_candidate {
    uint32_t tgt, hits, win_beg, win_end;
};

}  // extern "C"

namespace {

bool cand_before(const or_candidate& a, const or_candidate& b) {  // S12
    if (a.hits != b.hits) return a.hits > b.hits;
    return a.tgt < b.tgt;
}

// ---- §4.2, §5.6 P:771-786, S11-S13: top hits of ONE partition ----
// `locs` is the accumulated (unsorted) location list; the oracle sorts it,
// builds the window-count statistic and, for every target, scans every begin
// window b among its hit windows for the sum over [b, b+sws-1] (brute force).
std::vector<or_candidate> top_hits(std::vector<uint64_t> locs, uint32_t sws, uint32_t m) {
    std::sort(locs.begin(), locs.end());                       // step (6)
    std::map<uint32_t, std::map<uint32_t, uint32_t>> counts;   // step (7): t -> j -> hits
    for (uint64_t l : locs) counts[(uint32_t)(l >> 32)][(uint32_t)l] += 1;
    std::vector<or_candidate> best_per_target;                 // step (8)
    for (auto& [t, wins] : counts) {
        or_candidate best{t, 0, 0, 0};
        bool have = false;
        for (auto& [b, c0] : wins) {
            (void)c0;
            uint64_t last = (uint64_t)b + sws - 1;
            uint32_t hits = 0, end = b;
            for (auto& [j, c] : wins)
                if (j >= b && (uint64_t)j <= last) { hits += c; end = std::max(end, j); }
            if (!have || hits > best.hits) {  // strict '>' keeps the smallest b (S11)
                best = {t, hits, b, end};
                have = true;
            }
        }
        if (have) best_per_target.push_back(best);
    }
    std::sort(best_per_target.begin(), best_per_target.end(), cand_before);
    if (best_per_target.size() > m) best_per_target.resize(m);
    return best_per_target;
}

}  // namespace

extern "C" {

// Expose the per-partition top-hit step for the Figure 1 pin.
uint32_t or_top_hits(uint64_t n, const uint64_t* locs, uint32_t sws, uint32_t m, or_candidate* out) {
    std::vector<uint64_t> v(locs, locs + n);
    auto c = top_hits(v, sws, m);
    for (size_t i = 0; i < c.size(); ++i) out[i] = c[i];
    return (uint32_t)c.size();
}

// ---- P:609-618, Fig. 1 P:412-418 vs P:390-394, S12/S13: partition merge ----
uint32_t or_merge_candidates(uint32_t n_lists, uint32_t m, const or_candidate* lists,
                             const uint32_t* list_sizes, or_candidate* out) {
    std::vector<or_candidate> all;
    for (uint32_t i = 0; i < n_lists; ++i)
        for (uint32_t j = 0; j < list_sizes[i]; ++j) all.push_back(lists[i * m + j]);
    std::sort(all.begin(), all.end(), cand_before);
    if (all.size() > m) all.resize(m);
    for (size_t i = 0; i < all.size(); ++i) out[i] = all[i];
    return (uint32_t)all.size();
}

}  // extern "C"

namespace {

// ---- §4.2: taxonomy + LCA by naive parent walks -------------
struct Taxonomy {
    std::vector<uint32_t> parent;  // id 0 invalid; root.parent == root
    uint32_t lca(uint32_t a, uint32_t b) const {
        if (a == 0) return b;
        if (b == 0) return a;
        std::set<uint32_t> anc;
        for (uint32_t x = a;; x = parent[x]) {
            anc.insert(x);
            if (parent[x] == x) break;
        }
        for (uint32_t y = b;; y = parent[y]) {
            if (anc.count(y)) return y;
            if (parent[y] == y) break;
        }
        return 0;  // disconnected forest: no common ancestor
    }
};

struct Db {
    or_sketch_params sp{};
    uint32_t cap = 254, m = 4, hits_min = 5, hits_diff = 4, P = 1;
    uint64_t insert_size_max = 0;  // reading S25 (0: S10 only)
    Taxonomy tax;
    std::vector<std::map<uint32_t, std::vector<uint64_t>>> parts;  // D1/D3: feature -> locations
    std::map<uint32_t, uint32_t> taxon_of;                          // target id -> taxon
    std::vector<uint64_t> running_bp;
    bool finalized = false;
    bool filter_on = false;
    std::set<uint32_t> filter;  // feature-restricted oracle
};

}  // namespace

extern "C" {

void* or_db_create(uint32_t k, uint32_t s, uint32_t w, uint32_t cap, uint32_t m, uint32_t hits_min,
                   uint32_t hits_diff, uint32_t P, uint32_t n_taxa, const uint32_t* parent) {
    Db* db = new Db();
    db->sp = {k, s, w, 1u, nullptr};
    db->cap = cap;
    db->m = m;
    db->hits_min = hits_min;
    db->hits_diff = hits_diff;
    db->P = P;
    db->tax.parent.assign(parent, parent + n_taxa);
    db->parts.resize(P);
    db->running_bp.assign(P, 0);
    return db;
}

void or_db_destroy(void* h) { delete (Db*)h; }

// Restrict stored locations to a feature set (exact for reads whose features
// all lie in the set).
void or_db_set_feature_filter(void* h, uint64_t n, const uint32_t* feats) {
    Db* db = (Db*)h;
    db->filter_on = true;
    db->filter.insert(feats, feats + n);
}

// ---- §4.1 P:441-443 (build): every sketch feature of window j of target t is
// inserted with location (t, j) into its partition's map (S20: (t<<32)|j).
// partition_ids == NULL -> S9 greedy rule.  Returns 0 or -1 on bad input.
int or_db_insert(void* h, uint32_t n, const char* seqs, const uint64_t* offsets, const uint32_t* ids,
                 const uint32_t* taxa, const uint32_t* partition_ids) {
    Db* db = (Db*)h;
    if (db->finalized) return -1;
    std::vector<uint32_t> part(n);
    if (partition_ids) {  // S9: explicitly placed targets count towards their partition's bp too
        part.assign(partition_ids, partition_ids + n);
        for (uint32_t i = 0; i < n; ++i) db->running_bp[part[i]] += offsets[i + 1] - offsets[i];
    } else {
        std::vector<uint64_t> lens(n);
        for (uint32_t i = 0; i < n; ++i) lens[i] = offsets[i + 1] - offsets[i];
        or_plan_partitions(db->P, n, lens.data(), db->running_bp.data(), part.data());
    }
    for (uint32_t i = 0; i < n; ++i) {
        if (db->taxon_of.count(ids[i])) return -1;
        db->taxon_of[ids[i]] = taxa[i];
        std::string seq(seqs + offsets[i], seqs + offsets[i + 1]);
        auto sk = sketch_sequence(db->sp, seq);
        for (size_t j = 0; j < sk.size(); ++j)
            for (uint32_t f : sk[j]) {
                if (db->filter_on && !db->filter.count(f)) continue;
                db->parts[part[i]][f].push_back(((uint64_t)ids[i] << 32) | (uint64_t)j);
            }
    }
    return 0;
}

// Feature-restricted build at full workload size.  The
// targets' sketches are independent, so `threads` host threads each sketch a
// strided share of the targets with the same sketch_sequence as
// or_db_insert and keep only the filtered features; the kept locations are
// then appended target by target in insertion order, exactly as or_db_insert
// would.  Requires a feature filter (the full map would not fit).
int or_db_insert_restricted(void* h, uint32_t n, const char* seqs, const uint64_t* offsets, const uint32_t* ids,
                            const uint32_t* taxa, const uint32_t* partition_ids, uint32_t threads) {
    Db* db = (Db*)h;
    if (db->finalized || !db->filter_on || threads == 0) return -1;
    std::vector<uint32_t> part(n);
    if (partition_ids) {  // S9: explicitly placed targets count towards their partition's bp too
        part.assign(partition_ids, partition_ids + n);
        for (uint32_t i = 0; i < n; ++i) db->running_bp[part[i]] += offsets[i + 1] - offsets[i];
    } else {
        std::vector<uint64_t> lens(n);
        for (uint32_t i = 0; i < n; ++i) lens[i] = offsets[i + 1] - offsets[i];
        or_plan_partitions(db->P, n, lens.data(), db->running_bp.data(), part.data());
    }
    // per target: (feature, window) pairs in window order, filtered
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> kept(n);
    auto work = [&](uint32_t t0) {
        for (uint32_t i = t0; i < n; i += threads) {
            std::string seq(seqs + offsets[i], seqs + offsets[i + 1]);
            auto sk = sketch_sequence(db->sp, seq);
            for (size_t j = 0; j < sk.size(); ++j)
                for (uint32_t f : sk[j])
                    if (db->filter.count(f)) kept[i].push_back({f, (uint32_t)j});
        }
    };
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    for (uint32_t i = 0; i < n; ++i) {
        if (db->taxon_of.count(ids[i])) return -1;
        db->taxon_of[ids[i]] = taxa[i];
        for (auto& [f, j] : kept[i]) db->parts[part[i]][f].push_back(((uint64_t)ids[i] << 32) | (uint64_t)j);
    }
    return 0;
}

// ---- P:465-466 + S7: per (feature, partition) keep the `cap` smallest (t,j).
void or_db_finalize(void* h) {
    Db* db = (Db*)h;
    for (auto& part : db->parts)
        for (auto& [f, v] : part) {
            std::sort(v.begin(), v.end());
            if (v.size() > db->cap) v.resize(db->cap);
        }
    db->finalized = true;
}

// Sorted location list of one feature in one partition.
uint32_t or_db_feature_locations(void* h, uint32_t p, uint32_t f, uint64_t* out, uint32_t out_cap) {
    Db* db = (Db*)h;
    auto it = db->parts[p].find(f);
    if (it == db->parts[p].end()) return 0;
    uint32_t n = (uint32_t)it->second.size();
    for (uint32_t i = 0; i < n && i < out_cap; ++i) out[i] = it->second[i];
    return n;
}

// Dump a partition in key order: keys[n_keys], counts[n_keys], values[n_values].
// Pass NULL buffers to query sizes.
void or_db_dump_partition(void* h, uint32_t p, uint32_t* keys, uint32_t* counts, uint64_t* values,
                          uint64_t* n_keys, uint64_t* n_values) {
    Db* db = (Db*)h;
    uint64_t nk = 0, nv = 0;
    for (auto& [f, v] : db->parts[p]) {
        if (keys) keys[nk] = f;
        if (counts) counts[nk] = (uint32_t)v.size();
        for (uint64_t x : v) {
            if (values) values[nv] = x;
            ++nv;
        }
        ++nk;
    }
    *n_keys = nk;
    *n_values = nv;
}

uint32_t or_lca(void* h, uint32_t a, uint32_t b) { return ((Db*)h)->tax.lca(a, b); }

// ---- §4.2 P:598-603 + S15/S16: classification of one record ---------------
uint32_t or_classify_candidates(void* h, uint32_t n, const or_candidate* c) {
    Db* db = (Db*)h;
    if (n == 0 || c[0].hits < db->hits_min) return 0;  // S23: 0 = unclassified
    uint32_t taxon = 0;
    uint32_t in_s = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (c[0].hits - c[i].hits > db->hits_diff) continue;
        uint32_t t = db->taxon_of.at(c[i].tgt);
        taxon = in_s == 0 ? t : db->tax.lca(taxon, t);
        ++in_s;
    }
    return taxon;
}

// sws reading S10: 2 + floor((|r1|+|r2|)/stride).
// Reading S25 (insertSizeMax-style): a PAIRED record
// (mate present) uses max(|r1|+|r2|, insert_size_max) as its span.
uint32_t or_sws(void* h, uint64_t len1, uint64_t len2, int paired) {
    Db* db = (Db*)h;
    uint64_t stride = db->sp.w - db->sp.k + 1;
    uint64_t span = len1 + len2;
    if (paired && db->insert_size_max > span) span = db->insert_size_max;
    return (uint32_t)(2 + span / stride);
}

void or_db_set_insert_size_max(void* h, uint64_t v) { ((Db*)h)->insert_size_max = v; }

// ---- §4.2, Fig. 1: classify read records -------------------------
// out_cand: n_reads*m candidates (tgt==UINT32_MAX pads).  out_part_cand
// (nullable): n_reads*P*m per-partition lists.  out_n_locs (nullable):
// n_reads*P accumulated location counts (diagnostic).
static void classify_range(void* h, uint64_t r_begin, uint64_t r_end, const char* reads, const uint64_t* read_offsets,
                           const char* mates, const uint64_t* mate_offsets, uint32_t* out_taxon, or_candidate* out_cand,
                           or_candidate* out_part_cand, uint64_t* out_n_locs) {
    Db* db = (Db*)h;
    const uint32_t m = db->m;
    for (uint64_t r = r_begin; r < r_end; ++r) {
        std::string r1(reads + read_offsets[r], reads + read_offsets[r + 1]);
        std::string r2;
        if (mates) r2.assign(mates + mate_offsets[r], mates + mate_offsets[r + 1]);
        // S17/S18: sketch each mate's windows separately; keep duplicates.
        std::vector<uint32_t> F;
        for (auto& sk : sketch_sequence(db->sp, r1)) F.insert(F.end(), sk.begin(), sk.end());
        for (auto& sk : sketch_sequence(db->sp, r2)) F.insert(F.end(), sk.begin(), sk.end());
        uint32_t sws = or_sws(h, r1.size(), r2.size(), mates != nullptr);
        std::vector<or_candidate> lists(db->P * m, or_candidate{0xFFFFFFFFu, 0, 0, 0});
        std::vector<uint32_t> sizes(db->P, 0);
        for (uint32_t p = 0; p < db->P; ++p) {
            std::vector<uint64_t> L;  // query every feature, collect lists
            for (uint32_t f : F) {
                auto it = db->parts[p].find(f);
                if (it != db->parts[p].end()) L.insert(L.end(), it->second.begin(), it->second.end());
            }
            if (out_n_locs) out_n_locs[r * db->P + p] = L.size();
            auto c = top_hits(L, sws, m);
            sizes[p] = (uint32_t)c.size();
            for (size_t i = 0; i < c.size(); ++i) lists[p * m + i] = c[i];
        }
        if (out_part_cand)
            for (uint32_t i = 0; i < db->P * m; ++i) out_part_cand[r * db->P * m + i] = lists[i];
        std::vector<or_candidate> merged(m);
        uint32_t nm = or_merge_candidates(db->P, m, lists.data(), sizes.data(), merged.data());
        for (uint32_t i = 0; i < m; ++i)
            out_cand[r * m + i] = i < nm ? merged[i] : or_candidate{0xFFFFFFFFu, 0, 0, 0};
        out_taxon[r] = or_classify_candidates(h, nm, merged.data());
    }
}

int or_classify(void* h, uint64_t n_reads, const char* reads, const uint64_t* read_offsets, const char* mates,
                const uint64_t* mate_offsets, uint32_t* out_taxon, or_candidate* out_cand,
                or_candidate* out_part_cand, uint64_t* out_n_locs) {
    Db* db = (Db*)h;
    if (!db->finalized) return -1;
    classify_range(h, 0, n_reads, reads, read_offsets, mates, mate_offsets, out_taxon, out_cand, out_part_cand,
                   out_n_locs);
    return 0;
}

// The same query phase on `threads` host threads (SURVEY §8(d) "Oracle
// timing": the finalized maps are read-only, so records are independent);
// thread t classifies the contiguous record slice [t n / T, (t + 1) n / T).
// Results are identical to or_classify's.
int or_classify_threads(void* h, uint64_t n_reads, const char* reads, const uint64_t* read_offsets,
                        const char* mates, const uint64_t* mate_offsets, uint32_t* out_taxon, or_candidate* out_cand,
                        uint32_t threads) {
    Db* db = (Db*)h;
    if (!db->finalized || threads == 0) return -1;
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t)
        pool.emplace_back(classify_range, h, n_reads * t / threads, n_reads * (t + 1) / threads, reads, read_offsets,
                          mates, mate_offsets, out_taxon, out_cand, nullptr, nullptr);
    for (auto& th : pool) th.join();
    return 0;
}

}  // extern "C"
