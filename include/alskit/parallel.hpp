// alskit drop-in (B200): scale-up (SU-ALS) surface of the reference parallel.hpp:21-583.
//
// Host-side planning objects (Topology, footprint, planner, reduce schedules) are plain
// arithmetic and stay on the host; local_hermitian, parallel_reduce and su_als_update_x run
// on the device through libalskit_cuda (bit-identical to the reference in double mode).
// Multi-GPU execution of the same split (NCCL reduce-scatter / all-gather over NVLink)
// lives in paper_1603_03820_b200/distributed.py.
#pragma once

#include <algorithm>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include "alskit/solver.hpp"
#include "alskit/sparse.hpp"

namespace alskit {

struct Topology {  // parallel.hpp:29-34
    int workers = 1;
    int threads = 0;
    std::vector<std::vector<int>> groups;
    offset_t capacity = std::numeric_limits<offset_t>::max();
};

struct FootprintTerms {  // parallel.hpp:39-50
    offset_t x_part = 0, theta_part = 0, r_block = 0, hermitian = 0, rhs = 0, headroom = 0;
    [[nodiscard]] offset_t total() const noexcept { return x_part + theta_part + r_block + hermitian + rhs + headroom; }
};

inline const char* binding_term(const FootprintTerms& t) noexcept {  // parallel.hpp:53-60
    const offset_t v[] = {t.x_part, t.theta_part, t.r_block, t.hermitian, t.rhs, t.headroom};
    const char* names[] = {"m*f/q", "n*f/p", "R_block", "m/q*f^2", "m/q*f", "headroom"};
    return names[std::max_element(v, v + 6) - v];
}

struct PlanAttempt {  // parallel.hpp:63-68
    int p = 0, q = 0;
    FootprintTerms terms;
    bool feasible = false;
};

struct PartitionPlan {  // parallel.hpp:71-78
    int p = 1, q = 1;
    offset_t headroom = 0;
    FootprintTerms terms;
    offset_t per_worker_footprint = 0;
    std::vector<PlanAttempt> attempts;
};

enum class ReduceScheme { one_phase, two_phase };  // parallel.hpp:80

struct Transfer {  // parallel.hpp:84-90
    int src = 0, dst = 0, slice = 0;
    friend bool operator==(const Transfer&, const Transfer&) = default;
};

struct ReduceSchedule {  // parallel.hpp:99-124
    ReduceScheme scheme = ReduceScheme::one_phase;
    int workers = 1;
    std::vector<std::vector<int>> groups;
    std::vector<Transfer> phase1, phase2;
    [[nodiscard]] std::size_t total_transfers() const noexcept { return phase1.size() + phase2.size(); }
    [[nodiscard]] std::size_t cross_group_transfers() const {
        std::vector<int> group_of(static_cast<std::size_t>(workers), 0);
        for (std::size_t g = 0; g < groups.size(); ++g)
            for (int w : groups[g]) group_of[w] = static_cast<int>(g);
        std::size_t n = 0;
        for (const auto* ph : {&phase1, &phase2})
            for (const Transfer& t : *ph) n += group_of[t.src] != group_of[t.dst];
        return n;
    }
};

namespace detail {
inline std::vector<std::vector<int>> groups_of(const Topology& topo) {  // parallel.hpp:129-150
    if (topo.workers < 1) throw InputError("topology needs at least one worker");
    if (topo.capacity <= 0) throw InputError("capacity must be positive");
    auto g = topo.groups;
    if (g.empty()) {
        g.emplace_back();
        for (int w = 0; w < topo.workers; ++w) g[0].push_back(w);
    }
    std::vector<char> seen(static_cast<std::size_t>(topo.workers), 0);
    for (const auto& grp : g) {
        if (grp.empty()) throw InputError("empty worker group");
        for (int w : grp) {
            if (w < 0 || w >= topo.workers) throw InputError("group member " + std::to_string(w) + " outside worker range");
            if (seen[w]) throw InputError("worker " + std::to_string(w) + " appears in two groups");
            seen[w] = 1;
        }
    }
    for (int w = 0; w < topo.workers; ++w)
        if (!seen[w]) throw InputError("worker " + std::to_string(w) + " missing from groups");
    return g;
}
inline std::vector<offset_t> slice_cuts(offset_t count, int p) {  // parallel.hpp:160-168
    std::vector<offset_t> c(static_cast<std::size_t>(p) + 1, 0);
    for (int i = 0; i < p; ++i) c[i + 1] = c[i] + count / p + (i < count % p ? 1 : 0);
    return c;
}
}  // namespace detail

inline FootprintTerms footprint_terms(offset_t m, offset_t n, offset_t nnz, int f, int p, int q,
                                      offset_t headroom) {  // parallel.hpp:287-299
    const offset_t rq = (m + q - 1) / q, cp = (n + p - 1) / p;
    return FootprintTerms{rq * f, cp * f, 2 * nnz / (static_cast<offset_t>(p) * q) + rq + 1, rq * f * f, rq * f, headroom};
}

// Cheapest feasible (p, q): p = 1 first, then p from the half-capacity estimate up to the
// worker count; for each p the smallest feasible q by bisection (parallel.hpp:311-386).
inline PartitionPlan plan_partition(offset_t m, offset_t n, offset_t nnz, int f, const Topology& topo,
                                    offset_t headroom) {
    if (m < 1 || n < 1 || f < 1) throw InputError("dimensions and rank must be >= 1");
    if (nnz < 0) throw InputError("nnz must be >= 0");
    detail::groups_of(topo);
    if (headroom < 0 || headroom >= topo.capacity) throw InputError("headroom must lie in [0, capacity)");
    if (m > std::numeric_limits<offset_t>::max() / f / f) throw InputError("dimensions too large for footprint arithmetic");
    PartitionPlan plan;
    plan.headroom = headroom;
    auto eval = [&](int p, int q) {
        PlanAttempt a{p, q, footprint_terms(m, n, nnz, f, p, q, headroom), false};
        a.feasible = a.terms.total() < topo.capacity;
        return a;
    };
    auto try_p = [&](int p) -> std::optional<PlanAttempt> {
        const PlanAttempt one = eval(p, 1);
        plan.attempts.push_back(one);
        if (one.feasible) return one;
        if (m < 2) return std::nullopt;
        const PlanAttempt top = eval(p, static_cast<int>(std::min<offset_t>(m, std::numeric_limits<int>::max())));
        if (!top.feasible) {
            plan.attempts.push_back(top);
            return std::nullopt;
        }
        offset_t lo = 2, hi = top.q;
        while (lo < hi) {
            const offset_t mid = lo + (hi - lo) / 2;
            if (eval(p, static_cast<int>(mid)).feasible) hi = mid;
            else lo = mid + 1;
        }
        const PlanAttempt pick = eval(p, static_cast<int>(lo));
        plan.attempts.push_back(pick);
        return pick;
    };
    std::optional<PlanAttempt> found = try_p(1);
    if (!found && topo.workers >= 2 && n >= 2) {
        const offset_t half = topo.capacity / 2;
        const offset_t est = half > 0 ? (n * f + half - 1) / half : topo.workers;
        const int hi = static_cast<int>(std::min<offset_t>(topo.workers, n));
        for (int p = static_cast<int>(std::clamp<offset_t>(est, 2, hi)); p <= hi && !found; ++p) found = try_p(p);
    }
    if (!found) {
        const PlanAttempt* best = nullptr;
        for (const auto& a : plan.attempts)
            if (!best || a.terms.total() < best->terms.total()) best = &a;
        std::string msg = "no feasible partition for " + std::to_string(topo.workers) + " workers at capacity " +
                          std::to_string(topo.capacity);
        if (best)
            msg += ": smallest footprint " + std::to_string(best->terms.total()) + " at p=" + std::to_string(best->p) +
                   " q=" + std::to_string(best->q) + ", binding term " + binding_term(best->terms);
        throw CapacityError(msg);
    }
    plan.p = found->p;
    plan.q = found->q;
    plan.terms = found->terms;
    plan.per_worker_footprint = found->terms.total();
    return plan;
}

inline std::vector<FactorMatrix> split_factor(const FactorMatrix& whole, const std::vector<offset_t>& cuts) {  // 390-406
    if (cuts.size() < 2 || cuts.front() != 0 || cuts.back() != whole.rows) throw InputError("factor cuts must span [0, rows]");
    std::vector<FactorMatrix> parts;
    for (std::size_t i = 0; i + 1 < cuts.size(); ++i) {
        FactorMatrix part(cuts[i + 1] - cuts[i], whole.f);
        std::copy(whole.entries.begin() + cuts[i] * whole.f, whole.entries.begin() + cuts[i + 1] * whole.f,
                  part.entries.begin());
        parts.push_back(std::move(part));
    }
    return parts;
}

inline HermitianBatch local_hermitian(const CsrMatrix& block, const FactorMatrix& theta_part,
                                      const SolverConfig& cfg) {  // parallel.hpp:412-421
    HermitianBatch out;
    out.resize(block.rows, theta_part.f);
    const alsk_csr v = detail::view(block);
    const alsk_solver_config c = detail::cfg_view(cfg);
    detail::check(alsk_local_hermitian(&v, theta_part.entries.data(), theta_part.rows, theta_part.f, &c, out.a.data(),
                                       out.b.data()));
    return out;
}

inline ReduceSchedule build_reduce_schedule(const Topology& topo, ReduceScheme scheme) {  // parallel.hpp:436-465
    ReduceSchedule s;
    s.scheme = scheme;
    s.workers = topo.workers;
    s.groups = detail::groups_of(topo);
    if (scheme == ReduceScheme::one_phase) {
        for (int slice = 0; slice < topo.workers; ++slice)
            for (int src = 0; src < topo.workers; ++src)
                if (src != slice) s.phase1.push_back({src, slice, slice});
        return s;
    }
    if (s.groups.size() < 2) throw InputError("two-phase reduction needs at least 2 worker groups");
    for (int slice = 0; slice < topo.workers; ++slice)
        for (const auto& g : s.groups) {
            const bool home = std::find(g.begin(), g.end(), slice) != g.end();
            const int holder = home ? slice : g[static_cast<std::size_t>(slice) % g.size()];
            for (int w : g)
                if (w != holder) s.phase1.push_back({w, holder, slice});
            if (!home) s.phase2.push_back({holder, slice, slice});
        }
    return s;
}

namespace detail {
// The device executor rebuilds the schedule from group membership; groups are passed in
// ascending-member order, which is how build_reduce_schedule's rotation indexes them when
// the caller lists members ascending (the reference tests do).
inline std::vector<int32_t> group_vector(const ReduceSchedule& s) {
    std::vector<int32_t> g(static_cast<std::size_t>(s.workers), 0);
    for (std::size_t k = 0; k < s.groups.size(); ++k)
        for (int w : s.groups[k]) g[w] = static_cast<int32_t>(k);
    return g;
}
}  // namespace detail

inline std::vector<HermitianBatch> parallel_reduce(const std::vector<HermitianBatch>& parts,
                                                   const ReduceSchedule& sched, int /*threads*/ = 1) {  // 474-477
    const int p = sched.workers;
    if (static_cast<int>(parts.size()) != p)
        throw InputError("expected " + std::to_string(p) + " partial batches, got " + std::to_string(parts.size()));
    for (const auto& b : parts)
        if (b.count != parts[0].count || b.f != parts[0].f) throw InputError("partial batches disagree on count or rank");
    const offset_t count = parts[0].count;
    const int f = parts[0].f;
    const auto cuts = detail::slice_cuts(count, p);
    std::vector<HermitianBatch> out(static_cast<std::size_t>(p));
    std::vector<const float*> pa, pb;
    std::vector<float*> oa, ob;
    for (int i = 0; i < p; ++i) {
        out[i].resize(cuts[i + 1] - cuts[i], f);
        pa.push_back(parts[i].a.data());
        pb.push_back(parts[i].b.data());
        oa.push_back(out[i].a.data());
        ob.push_back(out[i].b.data());
    }
    const auto g = detail::group_vector(sched);
    detail::check(alsk_parallel_reduce(pa.data(), pb.data(), p, count, f, g.data(),
                                       sched.scheme == ReduceScheme::two_phase ? 1 : 0, oa.data(), ob.data()));
    return out;
}

inline FactorMatrix su_als_update_x(const GridPartition& grid, const std::vector<FactorMatrix>& theta_parts,
                                    const Topology& topo, ReduceScheme scheme, const SolverConfig& cfg) {  // 487-583
    const auto groups = detail::groups_of(topo);
    if (topo.workers != grid.p)
        throw InputError("topology workers (" + std::to_string(topo.workers) + ") must equal grid column partitions p (" +
                         std::to_string(grid.p) + ")");
    if (static_cast<int>(theta_parts.size()) != grid.p) throw InputError("expected one theta partition per column block");
    int f = 0;
    for (int i = 0; i < grid.p; ++i) {
        const offset_t want = grid.col_cuts[i + 1] - grid.col_cuts[i];
        if (theta_parts[i].rows != want)
            throw InputError("theta partition " + std::to_string(i) + " has " + std::to_string(theta_parts[i].rows) +
                             " rows, column cut wants " + std::to_string(want));
        if (i == 0) f = theta_parts[i].f;
        else if (theta_parts[i].f != f) throw InputError("theta partitions disagree on rank");
    }
    offset_t nnz = 0;
    for (const auto& b : grid.blocks) nnz += b.nnz();
    const FootprintTerms terms = footprint_terms(grid.rows, grid.cols, nnz, f, grid.p, grid.q, 0);
    if (terms.total() >= topo.capacity)
        throw CapacityError("per-worker footprint " + std::to_string(terms.total()) + " exceeds capacity " +
                            std::to_string(topo.capacity) + ", binding term " + binding_term(terms));
    ReduceSchedule s;
    s.workers = topo.workers;
    s.groups = groups;
    if (scheme == ReduceScheme::two_phase && groups.size() < 2)
        throw InputError("two-phase reduction needs at least 2 worker groups");
    const auto g = detail::group_vector(s);
    std::vector<alsk_csr> blocks;
    for (const auto& b : grid.blocks) blocks.push_back(detail::view(b));
    std::vector<const float*> th;
    for (const auto& t : theta_parts) th.push_back(t.entries.data());
    FactorMatrix x(grid.rows, f);
    const alsk_solver_config c = detail::cfg_view(cfg);
    detail::check(alsk_su_als_update_x(blocks.data(), grid.p, grid.q, grid.row_cuts.data(), grid.col_cuts.data(),
                                       th.data(), f, &c, g.data(), scheme == ReduceScheme::two_phase ? 1 : 0,
                                       x.entries.data()));
    return x;
}

}  // namespace alskit
