// plan.cpp -- see plan.h.  Canonical ordering rules (readings R8, R10):
//   groups = distinct adapter ids >= 0 that own >= 1 token, ascending id;
//   tokens ascending within a group; pages in rank order;
//   seg_kind = PREFILL if id >= 0 and len >= L_tc, DECODE if id >= 0 and 1 <= len < L_tc, else NONE.
#include "plan.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernel_config.h"

#ifndef LORA_EXP_PF_SPLIT
#define LORA_EXP_PF_SPLIT 0
#endif
#ifndef LORA_EXP_PF_SPLITK
#define LORA_EXP_PF_SPLITK 0
#endif

namespace lora {

static inline int32_t f32_bits(float f) {
    int32_t b;
    std::memcpy(&b, &f, 4);
    return b;
}

static lora_status append_unit_table(Plan& pl, std::string& err);

lora_status build_plan(Plan& pl, const int32_t* ip, const int32_t* ids, int S, int H_in, int H_out,
                       int esz, int L_tc, bool tc_enabled, const AdapterTable& table, std::string& err,
                       int pad_zero_page, int pf_sms, int expand_budget) {
    if (S < 0) { err = "num_segments < 0"; return LORA_ERR_ARG; }
    if (S > 0 && (ip == nullptr || ids == nullptr)) { err = "seg_indptr/adapter_ids is NULL"; return LORA_ERR_ARG; }
    if (S > 0 && ip[0] != 0) { err = "seg_indptr[0] != 0"; return LORA_ERR_ARG; }
    // one hash lookup per segment (runs of one id reuse it); the records are used below
    static thread_local std::vector<const AdapterRec*> seg_rec;
    seg_rec.assign(S, nullptr);
    for (int i = 0; i < S; ++i) {
        if (ip[i + 1] < ip[i]) { err = "seg_indptr not non-decreasing at segment " + std::to_string(i); return LORA_ERR_ARG; }
        if (ids[i] >= 0) {
            if (i > 0 && ids[i] == ids[i - 1]) {
                seg_rec[i] = seg_rec[i - 1];
                continue;
            }
            auto it = table.find(ids[i]);
            if (it == table.end()) {
                err = "adapter_ids[" + std::to_string(i) + "] = " + std::to_string(ids[i]) + " is not loaded";
                return LORA_ERR_UNKNOWN_ADAPTER;
            }
            seg_rec[i] = &it->second;
        }
    }
    const int T = S > 0 ? ip[S] : 0;
    pl.reset();
    pl.T = T; pl.S = S; pl.L_tc = L_tc;

    // M1 token -> segment
    pl.tok_seg.resize(T);
    for (int i = 0; i < S; ++i)
        for (int t = ip[i]; t < ip[i + 1]; ++t) pl.tok_seg[t] = i;

    // M2 groups (ids >= 0 owning >= 1 token), ascending
    static thread_local std::vector<int32_t> gids;
    gids.clear();
    for (int i = 0; i < S; ++i)
        if (ids[i] >= 0 && ip[i + 1] > ip[i]) gids.push_back(ids[i]);
    std::sort(gids.begin(), gids.end());
    gids.erase(std::unique(gids.begin(), gids.end()), gids.end());
    const int G = (int)gids.size();
    pl.G = G;
    auto gidx = [&](int32_t id) { return (int)(std::lower_bound(gids.begin(), gids.end(), id) - gids.begin()); };

    // M5 seg kinds and M6 features
    pl.seg_kind.resize(S);
    static thread_local std::vector<int32_t> seg_group;
    seg_group.assign(S, -1);
    static thread_local std::vector<const AdapterRec*> group_rec;
    group_rec.assign(G, nullptr);
    for (int i = 0; i < S; ++i) {
        const int len = ip[i + 1] - ip[i];
        if (ids[i] < 0 || len == 0) { pl.seg_kind[i] = LORA_KIND_NONE; continue; }
        pl.seg_kind[i] = len >= L_tc ? LORA_KIND_PREFILL : LORA_KIND_DECODE;
        seg_group[i] = gidx(ids[i]);
        group_rec[seg_group[i]] = seg_rec[i];
        const int64_t r = seg_rec[i]->rank;
        pl.n_seg += 1;
        pl.max_rank = std::max(pl.max_rank, r);
        pl.sum_rank_seg += r;
        pl.sum_rank_tokens += r * len;
    }
    pl.nseg_x_maxrank = pl.n_seg * pl.max_rank;

    // M2/M3/M4 per-group tables
    pl.group_id = gids;
    pl.group_rank.resize(G); pl.group_scale.resize(G); pl.group_ntok.assign(G, 0);
    pl.group_page_off.resize(G); pl.group_tok_off.resize(G);
    for (int g = 0; g < G; ++g) {
        const AdapterRec& a = *group_rec[g];
        pl.group_rank[g] = a.rank;
        pl.group_scale[g] = a.scale;
        pl.group_page_off[g] = (int32_t)pl.pages.size();
        pl.pages.insert(pl.pages.end(), a.pages.begin(), a.pages.begin() + a.rank);
        pl.sum_rank_groups += a.rank;
    }
    for (int t = 0; t < T; ++t) {
        const int g = seg_group[pl.tok_seg[t]];
        if (g >= 0) pl.group_ntok[g] += 1;
    }
    int off = 0;
    for (int g = 0; g < G; ++g) { pl.group_tok_off[g] = off; off += pl.group_ntok[g]; }
    pl.group_tokens.resize(off);
    {
        std::vector<int32_t> fill(pl.group_tok_off);
        for (int t = 0; t < T; ++t) {
            const int g = seg_group[pl.tok_seg[t]];
            if (g >= 0) pl.group_tokens[fill[g]++] = t;
        }
    }

    // ---- kernel work ----
    // tokens of the SIMT path per group (ascending; flat, counting-sorted by group), and
    // tensor-core segments
    // tensor-core routing: PREFILL segments of rank <= kPfMaxRank while the tile records and
    // page lists fit the kernel-parameter blob; everything else takes the decode kernels
    static thread_local std::vector<uint8_t> on_tc;
    on_tc.assign(S, 0);
    if (tc_enabled) {
        std::vector<int32_t> group_pf_off(G, -1);
        std::vector<int32_t> pages_words;
        int tiles = 0;
        for (int i = 0; i < S; ++i) {
            const int g = seg_group[i];
            if (g < 0 || pl.seg_kind[i] != LORA_KIND_PREFILL || pl.group_rank[g] > kPfMaxRank) continue;
            const int len = ip[i + 1] - ip[i];
            const int nt = (len + 127) / 128;
            const int extra_pages = group_pf_off[g] < 0 ? pl.group_rank[g] : 0;
            if ((tiles + nt) * 8 + (int)pages_words.size() + extra_pages > kPfMaxBlobWords) continue;
            if (group_pf_off[g] < 0) {
                group_pf_off[g] = (int32_t)pages_words.size();
                pages_words.insert(pages_words.end(), pl.pages.begin() + pl.group_page_off[g],
                                   pl.pages.begin() + pl.group_page_off[g] + pl.group_rank[g]);
            }
            on_tc[i] = 1;
            tiles += nt;
            pl.prefill.push_back({ip[i], len, g});
        }
        // few token tiles (e.g. 70B prefill, 32 tiles): `split` CTAs per tile, each expanding a share
        // of the columns.  Split-K: the CTAs form a cluster (<= 8) that also splits the shrink's K,
        // exchanging fp32 partial D1 tiles through an L2 scratch (summed in rank order, deterministic)
        // -- nothing is read twice.  Used when <= 8 CTAs per tile are wanted or when the shrink
        // dominates (H_in > H_out); beyond 8 (very few tiles, e.g. one 512-token segment) the other
        // CTAs of a tile each recompute its shrink (column split; x re-read, mostly from L2).
        const int nct = H_out / 128;
        int split = 1;
        bool splitk = false;
        if (tiles > 0 && pf_sms > 0) {
            // experiment builds only (LORA_BUILD_DEFS): -DLORA_EXP_PF_SPLIT=s forces s CTAs per tile,
            // -DLORA_EXP_PF_SPLITK=1 forces the split-K cluster mode
            const int force_split = LORA_EXP_PF_SPLIT;
            split = force_split > 0 ? std::min(nct, force_split) : std::max(1, std::min(nct, pf_sms / tiles));
            splitk = LORA_EXP_PF_SPLITK || split <= 8 || H_in > H_out;
            if (splitk) split = std::min(split, std::min(8, H_in / 64));
            while (split > 1 && (tiles * split + (int)pages_words.size()) * 8 > kPfMaxBlobWords) --split;
        }
        pl.pf_cs = splitk ? split : 1;
        const int ctas = tiles * split;
        pl.n_pf_tiles = ctas;
        pl.n_prefill_tiles = tiles;
        pl.pf_blob.assign((size_t)ctas * 8 + pages_words.size(), 0);
        int tix = 0;
        for (const PrefillSeg& sg : pl.prefill) {
            for (int t0 = 0; t0 < sg.len; t0 += 128)
            for (int sp = 0; sp < split; ++sp) {
                int32_t* rec = pl.pf_blob.data() + (size_t)tix * 8;
                rec[6] = sp * nct / split;
                rec[7] = (sp + 1) * nct / split;
                rec[0] = sg.tok0 + t0;
                rec[1] = std::min(128, sg.len - t0);
                rec[2] = pl.group_rank[sg.group];
                rec[3] = ctas * 8 + group_pf_off[sg.group];
                rec[4] = f32_bits(pl.group_scale[sg.group]);
                // rec[5]: first page when the adapter's pages are one run (2D TMA boxes), else -1
                {
                    const int32_t* gp = pl.pages.data() + pl.group_page_off[sg.group];
                    bool run = true;
                    for (int j = 1; j < pl.group_rank[sg.group] && run; ++j) run = gp[j] == gp[0] + j;
                    rec[5] = run ? gp[0] : -1;
                }
                ++tix;
            }
        }
        std::copy(pages_words.begin(), pages_words.end(), pl.pf_blob.begin() + (size_t)ctas * 8);
    }
    static thread_local std::vector<int32_t> simt_off, simt_tok;
    simt_off.assign(G + 1, 0);
    for (int t = 0; t < T; ++t) {
        const int i = pl.tok_seg[t];
        const int g = seg_group[i];
        if (g >= 0 && !on_tc[i]) simt_off[g + 1] += 1;
    }
    for (int g = 0; g < G; ++g) simt_off[g + 1] += simt_off[g];
    simt_tok.resize(simt_off[G]);
    {
        static thread_local std::vector<int32_t> fill;
        fill.assign(simt_off.begin(), simt_off.end() - 1);
        for (int t = 0; t < T; ++t) {
            const int i = pl.tok_seg[t];
            const int g = seg_group[i];
            if (g >= 0 && !on_tc[i]) simt_tok[fill[g]++] = t;
        }
    }
    const int ksplit = ksplit_of(H_in, esz);
    // gc = (group, token chunk)
    struct Gc { int g, tok_off, ntok; };
    static thread_local std::vector<Gc> gcs;
    static thread_local std::vector<int32_t> blob_pages, blob_toks, group_blob_page, gp;
    gcs.clear();
    blob_pages.clear();
    blob_toks.clear();
    group_blob_page.assign(G, -1);
    for (int g = 0; g < G; ++g) {
        const int n_simt = simt_off[g + 1] - simt_off[g];
        if (n_simt == 0) continue;
        gp.assign(pl.pages.begin() + pl.group_page_off[g], pl.pages.begin() + pl.group_page_off[g] + pl.group_rank[g]);
        // padded-BGMV comparison mode (NEXT f4): every group's rank rows are padded to
        // the batch's max rank with the pool's all-zero page -- the work Punica's BGMV does
        if (pad_zero_page >= 0) gp.insert(gp.end(), (size_t)(pl.max_rank - pl.group_rank[g]), pad_zero_page);
        bool contiguous = true;
        for (size_t j = 1; j < gp.size() && contiguous; ++j) contiguous = gp[j] == gp[0] + (int32_t)j;
        if (contiguous) {
            group_blob_page[g] = ~gp[0];   // page reference ~first_page: no page words in the blob
        } else {
            group_blob_page[g] = (int32_t)blob_pages.size();
            blob_pages.insert(blob_pages.end(), gp.begin(), gp.end());
        }
        const int tc = tok_chunk(esz);
        const int32_t* st = simt_tok.data() + simt_off[g];
        for (int c = 0; c < n_simt; c += tc) {
            const int n = std::min(tc, n_simt - c);
            gcs.push_back({g, (int)blob_toks.size(), n});
            blob_toks.insert(blob_toks.end(), st + c, st + c + n);
        }
    }
    const int n_gc = (int)gcs.size();
    pl.n_gc = n_gc;
    pl.blob.assign(kHdrWords + kGcFields * n_gc + blob_pages.size() + blob_toks.size(), 0);
    int32_t* hdr = pl.blob.data();
    int32_t* gct = hdr + kHdrWords;
    const int pages_base = kHdrWords + kGcFields * n_gc;
    const int toks_base = pages_base + (int)blob_pages.size();
    int shrink = 0, expand = 0;
    int64_t voff = 0, vred = 0;
    // expand unit widths (DESIGN.md §6 N1).  expand_budget > 0: the widest units within that SMEM
    // budget (lora_apply_multi: kExpandSmemBudget, so a q/k/v grid is resident in one wave).  Single-
    // pool applies (expand_budget <= 0): round 1's power-of-two 32 KB units -- more, shorter CTAs --
    // while that grid is resident in one wave at >= 3 CTAs per SM, else the kExpandSmemBudget units.
    static thread_local std::vector<int32_t> gc_nc;
    gc_nc.resize(n_gc);
    auto size_units = [&](int budget) {
        int units = 0, smem = 0;
        for (int c = 0; c < n_gc; ++c) {
            const int r = pad_zero_page >= 0 ? (int)pl.max_rank : pl.group_rank[gcs[c].g];
            gc_nc[c] = expand_cols_gc(r, gcs[c].ntok, H_out, esz, budget);
            units += (H_out + gc_nc[c] - 1) / gc_nc[c];
            if (esz == 2) smem = std::max(smem, expand_mma_smem(r, gc_nc[c], gcs[c].ntok));
        }
        return std::make_pair(units, smem);
    };
    if (expand_budget > 0) {
        size_units(expand_budget);
    } else if (esz == 2) {
        const auto pw2 = size_units(0);
        const int sms = pf_sms > 0 ? pf_sms : 148;
        if (pw2.first > 3 * sms || pw2.second > kExpandSmemBudget3) size_units(kExpandSmemBudget);
    } else {
        size_units(0);
    }
    for (int c = 0; c < n_gc; ++c) {
        const int g = gcs[c].g, r = pad_zero_page >= 0 ? (int)pl.max_rank : pl.group_rank[g];
        int32_t* e = gct + kGcFields * c;
        e[GC_RANK] = r;
        e[GC_PAGE_OFF] = group_blob_page[g] < 0 ? group_blob_page[g] : pages_base + group_blob_page[g];
        e[GC_TOK_OFF] = toks_base + gcs[c].tok_off;
        e[GC_NTOK] = gcs[c].ntok;
        e[GC_SHRINK_BASE] = shrink;
        e[GC_EXPAND_BASE] = expand;
        e[GC_VOFF] = (int32_t)voff;
        e[GC_SCALE] = f32_bits(pl.group_scale[g]);
        e[GC_JOB] = 0;
        e[GC_VRED] = (int32_t)vred;
        const int nc = gc_nc[c];
        e[GC_NCOLS] = nc;
        shrink += ksplit * shrink_jblocks(r, esz);
        expand += (H_out + nc - 1) / nc;
        voff += (int64_t)ksplit * gcs[c].ntok * v_stride(r);
        vred += (int64_t)gcs[c].ntok * v_stride(r);
    }
    if (voff > INT32_MAX) { err = "batch too large for the SIMT scratch"; return LORA_ERR_ARG; }
    std::copy(blob_pages.begin(), blob_pages.end(), pl.blob.begin() + pages_base);
    std::copy(blob_toks.begin(), blob_toks.end(), pl.blob.begin() + toks_base);
    hdr[0] = n_gc; hdr[1] = shrink; hdr[2] = expand;
    hdr[3] = (int32_t)blob_pages.size(); hdr[4] = (int32_t)blob_toks.size(); hdr[5] = ksplit;
    pl.n_shrink = shrink; pl.n_expand = expand; pl.vbuf_floats = voff; pl.vred_floats = vred;
    pl.blob_esz = esz;
    return append_unit_table(pl, err);
}

// Appends the per-unit table (kernel_config.h): kUnitWords words per unit, shrink units first,
// {(gc << 16) | index of the unit in its gc, first page word of the unit, first token word of
// the gc, (rank << 16) | ntok}, so a CTA reads its whole work description with independent
// uniform parameter loads: one round trip, no search over the gc records, no dependent chain.
static lora_status append_unit_table(Plan& pl, std::string& err) {
    int32_t* h = pl.blob.data();
    const int n_gc = h[0], n_shrink = h[1], n_expand = h[2];
    if (n_gc >= (1 << 15)) { err = "too many (group, token-chunk) units"; return LORA_ERR_ARG; }
    if (pl.blob.size() >= ((size_t)1 << 19)) { err = "batch metadata too large"; return LORA_ERR_ARG; }
    const size_t base = pl.blob.size();
    // full 3-word records while the blob fits the kernel parameters, else 1 word per unit (the
    // kernels then read rank / tokens / pages from the gc record: one more dependent load)
    const size_t units = (size_t)n_shrink + n_expand;
// 3-word records only while the blob stays <= 16 KB of kernel parameters: a q/k/v lora_apply_multi of a
// c2 batch at 3 words (5,216 words, launched as 31.7 KB of parameters per grid) measured 117.7K vs
// 118.4K tok/s with 1-word records (2,552 words, 16 KB) -- the larger parameter block costs launch time
#ifndef LORA_UNIT_WORDS_MAX_BLOB
#define LORA_UNIT_WORDS_MAX_BLOB 4096
#endif
    const int uw = base + (size_t)kUnitWords * units <= (size_t)LORA_UNIT_WORDS_MAX_BLOB ? kUnitWords : 1;
    pl.unit_words = uw;
    pl.blob.resize(base + (size_t)uw * units);
    h = pl.blob.data();
    const int esz = pl.blob_esz;
    for (int c = 0; c < n_gc; ++c) {
        const int32_t* e = h + kHdrWords + kGcFields * c;
        const int s1 = c + 1 < n_gc ? e[kGcFields + GC_SHRINK_BASE] : n_shrink;
        const int e1 = c + 1 < n_gc ? e[kGcFields + GC_EXPAND_BASE] : n_expand;
        if (s1 - e[GC_SHRINK_BASE] > 0xffff || e1 - e[GC_EXPAND_BASE] > 0xffff) {
            err = "too many units per (group, token-chunk)";
            return LORA_ERR_ARG;
        }
        const int r = e[GC_RANK], njb = shrink_jblocks(r, esz);
        for (int u = e[GC_SHRINK_BASE]; u < s1; ++u) {
            const int local = u - e[GC_SHRINK_BASE];
            int32_t* w = h + base + (size_t)uw * u;
            w[0] = (c << 16) | local;
            if (uw == 1) continue;
            w[1] = page_ref_add(e[GC_PAGE_OFF], (local % njb) * shrink_rows(esz));
            w[2] = r | (e[GC_NTOK] << 9) | (e[GC_TOK_OFF] << 13);
        }
        for (int u = e[GC_EXPAND_BASE]; u < e1; ++u) {
            int32_t* w = h + base + (size_t)uw * (n_shrink + u);
            w[0] = (c << 16) | (u - e[GC_EXPAND_BASE]);
            if (uw == 1) continue;
            w[1] = e[GC_PAGE_OFF];
            w[2] = r | (e[GC_NTOK] << 9) | (e[GC_TOK_OFF] << 13);
        }
    }
    h[6] = (int32_t)base;
    pl.unit_tab = (int32_t)base;
    return LORA_OK;
}

lora_status merge_plans(const Plan* const* plans, int n, Plan& m, std::string& err) {
    m = Plan();
    if (n < 1 || n > kMaxJobs) { err = "between 1 and 4 pools per fused apply"; return LORA_ERR_ARG; }
    int n_gc = 0, n_pages = 0, n_toks = 0;
    for (int p = 0; p < n; ++p) {
        const int32_t* h = plans[p]->blob.data();
        if (plans[p]->blob.empty()) continue;
        n_gc += h[0];
        n_pages += h[3];
        n_toks += h[4];
    }
    m.blob.assign(kHdrWords + (size_t)kGcFields * n_gc + n_pages + n_toks, 0);
    const int pages_base = kHdrWords + kGcFields * n_gc, toks_base = pages_base + n_pages;
    int gc = 0, pg = 0, tk = 0, shrink = 0, expand = 0;
    int64_t voff = 0, vred = 0;
    for (int p = 0; p < n; ++p) {
        const Plan& q = *plans[p];
        if (q.blob.empty() || q.n_gc == 0) continue;
        const int32_t* h = q.blob.data();
        m.job_shrink_base[p] = shrink;
        m.job_expand_base[p] = expand;
        const int qpb = kHdrWords + kGcFields * h[0], qtb = qpb + h[3];
        for (int c = 0; c < h[0]; ++c) {
            const int32_t* e = h + kHdrWords + kGcFields * c;
            int32_t* o = m.blob.data() + kHdrWords + kGcFields * gc;
            for (int f = 0; f < kGcFields; ++f) o[f] = e[f];
            o[GC_PAGE_OFF] = e[GC_PAGE_OFF] < 0 ? e[GC_PAGE_OFF] : pages_base + pg + (e[GC_PAGE_OFF] - qpb);
            o[GC_TOK_OFF] = toks_base + tk + (e[GC_TOK_OFF] - qtb);
            o[GC_SHRINK_BASE] = e[GC_SHRINK_BASE] + shrink;
            o[GC_EXPAND_BASE] = e[GC_EXPAND_BASE] + expand;
            o[GC_VOFF] = (int32_t)(e[GC_VOFF] + voff);
            o[GC_VRED] = (int32_t)(e[GC_VRED] + vred);
            o[GC_JOB] = p;
            ++gc;
        }
        std::copy(h + qpb, h + qpb + h[3], m.blob.begin() + pages_base + pg);
        std::copy(h + qtb, h + qtb + h[4], m.blob.begin() + toks_base + tk);
        pg += h[3];
        tk += h[4];
        shrink += q.n_shrink;
        expand += q.n_expand;
        voff += q.vbuf_floats;
        vred += q.vred_floats;
    }
    if (voff > INT32_MAX) { err = "fused batch too large for the SIMT scratch"; return LORA_ERR_ARG; }
    int32_t* h = m.blob.data();
    h[0] = n_gc; h[1] = shrink; h[2] = expand; h[3] = n_pages; h[4] = n_toks; h[5] = 0;
    for (int p = 0; p < n; ++p)
        if (plans[p]->blob.empty() || plans[p]->n_gc == 0) {   // empty jobs own no units
            m.job_shrink_base[p] = p + 1 < n ? 0x7fffffff : 0x7fffffff;
            m.job_expand_base[p] = 0x7fffffff;
        }
    m.n_jobs = n;
    m.n_gc = n_gc;
    m.n_shrink = shrink;
    m.n_expand = expand;
    m.vbuf_floats = voff;
    m.vred_floats = vred;
    m.blob_esz = plans[0]->blob_esz;
    return append_unit_table(m, err);
}

}  // namespace lora
