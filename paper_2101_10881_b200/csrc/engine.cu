// Device engine: plan compilation, arena management, the layer scheduler and
// the C-ABI entry points that replace run_sequential / run_parallel /
// evaluate (proj/src/executor.cpp:168-276).
//
// Execution model. One grid launch per dependency level replaces the
// reference's barrier-per-phase thread pool (executor.cpp:185-231): conv
// layers, then the TermScale phase, then addition layers, then extraction.
// The launch sequence for a batch size is captured once into a CUDA graph
// and replayed, so a whole evaluation is a single graph launch.
//
// Plan-time rewrites (results stay bit-identical):
//  * In-place convolutions (the coefficient fold b_{n-2} := b_{n-2} * a,
//    jobgraph.cpp:115) are made out-of-place by versioning the slot: the
//    earlier job that produced the pre-fold value writes a scratch slot that
//    the fold (and any reader in between) reads instead. Every thread can
//    then stream its own coefficients without a block-wide input copy.
//  * Exponent folding (fold_exponents, jobgraph.cpp:168-197) becomes device
//    conv jobs in prologue layers (pse_evaluate only).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <memory>
#include <queue>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_graph.hpp"
#include "kernels.cuh"

namespace pse {
namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct ConvRow {
  int64_t in1, in2, out;
  uint8_t copy;
};

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return PSE_EINVAL;
  } catch (const CudaError& e) {
    set_error(e.what());
    return PSE_ECUDA;
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    return PSE_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return PSE_ESTATE;
  }
}

// stage: reference-layout static block [q][b][top][d+1] -> arena
__global__ void k_stage(const double* __restrict__ in, double* __restrict__ arena, Geom G, int64_t top, int batch,
                        int64_t in_point_words) {
  const int d1 = G.d + 1;
  const int64_t n = static_cast<int64_t>(G.Q) * batch * top * d1;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(t % d1);
    int64_t r = t / d1;
    const int64_t s = r % top;
    r /= top;
    const int64_t b = r % batch;
    const int q = static_cast<int>(r / batch);
    arena[b * G.point_words + s * G.slot_words + static_cast<int64_t>(q) * G.S + j] =
        in[(static_cast<int64_t>(q) * batch + b) * in_point_words + s * d1 + j];
  }
}

// exchange block of one rank: [point][i][slot_words] <-> arena slots
template <bool PACK>
__global__ void k_exchange(double* __restrict__ arena, double* __restrict__ buf, Geom G, const int* __restrict__ slots,
                           int count, int batch) {
  const int64_t n = static_cast<int64_t>(batch) * count * G.slot_words;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = t % G.slot_words;
    const int64_t r = t / G.slot_words;
    const int i = static_cast<int>(r % count);
    const int64_t b = r / count;
    double* a = arena + b * G.point_words + static_cast<int64_t>(slots[i]) * G.slot_words + w;
    if (PACK)
      buf[t] = *a;
    else
      *a = buf[t];
  }
}

// Peer gather (one polynomial sharded over devices): every slot rank r
// produced that the addition stage needs is copied from rank r's arena --
// peer memory over NVLink (CUDA IPC mapping) or the same device -- into this
// arena at the same offset (all ranks' arenas share the geometry). One launch
// for all peers: item = (peer list entry, point, word).
struct PeerList {
  const double* src;  // peer arena
  const int* slots;
  int count;
};
__global__ void k_gather_peers(double* __restrict__ arena, Geom G, const PeerList* __restrict__ peers, int npeers,
                               const int64_t* __restrict__ first1, int batch) {
  // first1[r]: words before peer entry r for ONE point; a batch scales it
  const int64_t n = first1[npeers] * batch;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int r = 0;
    while (t >= first1[r + 1] * batch) ++r;
    const int64_t u = t - first1[r] * batch;
    const int64_t w = u % G.slot_words;
    const int64_t rest = u / G.slot_words;
    const int i = static_cast<int>(rest % peers[r].count);
    const int64_t b = rest / peers[r].count;
    const int64_t off = b * G.point_words + static_cast<int64_t>(peers[r].slots[i]) * G.slot_words + w;
    arena[off] = peers[r].src[off];
  }
}

// arena -> reference DataArray layout [q][b][TS][d+1]
__global__ void k_export(const double* __restrict__ arena, double* __restrict__ out, Geom G, int64_t TS, int batch) {
  const int d1 = G.d + 1;
  const int64_t n = static_cast<int64_t>(G.Q) * batch * TS * d1;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(t % d1);
    int64_t r = t / d1;
    const int64_t s = r % TS;
    r /= TS;
    const int64_t b = r % batch;
    const int q = static_cast<int>(r / batch);
    out[t] = arena[b * G.point_words + s * G.slot_words + static_cast<int64_t>(q) * G.S + j];
  }
}

unsigned grid_for(int64_t n, int threads, int sms) {
  const int64_t need = (n + threads - 1) / threads;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sms) * 32)));
}

template <class T>
T* dev_alloc(size_t count) {
  void* p = nullptr;
  if (count == 0) return nullptr;
  ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

template <class T>
T* dev_upload(const std::vector<T>& v, cudaStream_t s) {
  T* p = dev_alloc<T>(v.size());
  if (p) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "upload");
  return p;
}

// Conv rows per layer (prologue layers first, then the graph's), with
// in-place jobs (out == in1, the coefficient fold b := b * a,
// jobgraph.cpp:115) made out-of-place: the earlier job that produced the
// pre-fold value writes a fresh slot (*next_slot++) that the fold and every
// reader in between read instead.
std::vector<std::vector<ConvRow>> versioned_layers(const pse_graph_desc& g,
                                                   const std::vector<std::vector<ConvRow>>& prologue,
                                                   int64_t* next_slot) {
  std::vector<std::vector<ConvRow>> layers = prologue;
  for (int32_t L = 0; L < g.n_conv_layers; ++L) {
    std::vector<ConvRow> rows;
    for (int64_t t = g.conv_layer_off[L]; t < g.conv_layer_off[L + 1]; ++t)
      rows.push_back({g.conv_in1[t], g.conv_in2[t], g.conv_out[t], g.conv_copy[t]});
    layers.push_back(std::move(rows));
  }
  std::map<int64_t, std::pair<size_t, size_t>> last_writer;  // slot -> (layer, row)
  for (size_t L = 0; L < layers.size(); ++L) {
    for (size_t r = 0; r < layers[L].size(); ++r) {
      ConvRow& j = layers[L][r];
      if (j.copy || j.out != j.in1) continue;
      auto it = last_writer.find(j.in1);
      if (it == last_writer.end()) throw std::invalid_argument("in-place job on a slot without an earlier writer");
      const int64_t s = j.in1, scratch = (*next_slot)++;
      const size_t Lw = it->second.first;
      layers[Lw][it->second.second].out = scratch;
      for (size_t L2 = Lw + 1; L2 <= L; ++L2)
        for (ConvRow& q : layers[L2]) {
          if (&q != &j && q.out == s && L2 < L) throw std::invalid_argument("slot rewritten before in-place use");
          if (q.in1 == s) q.in1 = scratch;
          if (!q.copy && q.in2 == s) q.in2 = scratch;
        }
    }
    for (size_t r = 0; r < layers[L].size(); ++r) last_writer[layers[L][r].out] = {L, r};
  }
  return layers;
}

// Banded conv schedule (see BandArgs in kernels.cuh), band width W. Tasks
// (job, band b, segment s <= b) -- one per band for copy jobs -- with the
// dependencies:
//   (J, b, s-1)                   the running sum of the same chains;
//   final band s of in1's job     steps i in segment s read x_i, i in band s;
//   final bands <= b of in2's job (segment 0; later segments read less);
// where "final band b" of a job is its task (b, b) (copy: its band-b task).
// Static inputs and outputs of earlier launches are ready from the start.
// Tasks are ranked by longest path to the exit. Wave mode: list-scheduled
// into waves of at most `cap_slots` 8-lane slots, one launch per wave. Flow
// mode: greedy list scheduling simulated in time gives the order in which
// the dataflow kernel hands out warp descriptors. Tasks are packed into
// descriptors of kSlots slots in that order (a task only joins the open
// descriptor if none of its dependencies is in it).
struct BandSched {
  std::vector<std::vector<int4>> waves;  // kSlots slots per warp descriptor, per wave
  std::vector<int> dep_off, deps;        // per descriptor (numbered in order): descriptors it waits for
  double makespan = 0;                   // flow: simulated, in steps (one step = one md_mul + md_add)
};

// ovh: fixed cost of a task (hand-out, dependency flags, partial sums) in steps
BandSched band_schedule(const std::vector<ConvRow>& rows, int d, int W, int64_t cap_slots, bool flow, int64_t procs,
                        double slack, double ovh) {
  const int nb = 1 + d / W;  // band 0 = [0, d % W + 1), then full bands (kernels.cuh)
  if (nb > 32767) throw std::invalid_argument("degree too large for the banded schedule");
  const int W0 = d % W + 1;
  auto lo = [&](int b) { return b == 0 ? 0 : W0 + (b - 1) * W; };
  const int nj = static_cast<int>(rows.size());
  std::map<int64_t, int> producer;
  for (int j = 0; j < nj; ++j) producer[rows[j].out] = j;
  std::vector<int64_t> base(nj + 1, 0);
  for (int j = 0; j < nj; ++j) base[j + 1] = base[j] + (rows[j].copy ? nb : nb * (nb + 1) / 2);
  const int64_t T = base[nj];
  if (T >= (int64_t(1) << 31)) throw std::invalid_argument("graph too large for the banded schedule");
  auto fin = [&](int j, int b) { return rows[j].copy ? base[j] + b : base[j] + b * (b + 1) / 2 + b; };
  std::vector<int> tjob(T);
  std::vector<int16_t> tb(T), ts(T);  // ts = -1: copy task
  std::vector<std::pair<int64_t, int64_t>> edges;
  for (int j = 0; j < nj; ++j) {
    const auto px = producer.find(rows[j].in1);
    const int X = px == producer.end() ? -1 : px->second;
    int Y = -1;
    if (!rows[j].copy) {
      const auto py = producer.find(rows[j].in2);
      Y = py == producer.end() ? -1 : py->second;
    }
    if (X >= j || Y >= j) throw std::logic_error("band schedule: jobs not in dependency order");
    for (int b = 0; b < nb; ++b) {
      if (rows[j].copy) {
        const int64_t t = base[j] + b;
        tjob[t] = j, tb[t] = b, ts[t] = -1;
        if (X >= 0) edges.emplace_back(fin(X, b), t);
        continue;
      }
      for (int s2 = 0; s2 <= b; ++s2) {
        const int64_t t = base[j] + b * (b + 1) / 2 + s2;
        tjob[t] = j, tb[t] = b, ts[t] = s2;
        if (s2 > 0) edges.emplace_back(t - 1, t);
        if (X >= 0) edges.emplace_back(fin(X, s2), t);
        if (s2 == 0 && Y >= 0)
          for (int b2 = 0; b2 <= b; ++b2) edges.emplace_back(fin(Y, b2), t);
      }
    }
  }
  // successor and predecessor lists (CSR); every edge goes from a lower to a
  // higher task id, so ids are a topological order
  std::vector<int64_t> off(T + 1, 0), succ(edges.size()), poff(T + 1, 0), pred(edges.size());
  std::vector<int> indeg(T, 0);
  for (auto& e : edges) ++off[e.first + 1], ++poff[e.second + 1], ++indeg[e.second];
  for (int64_t t = 0; t < T; ++t) off[t + 1] += off[t], poff[t + 1] += poff[t];
  {
    std::vector<int64_t> f1(off.begin(), off.end() - 1), f2(poff.begin(), poff.end() - 1);
    for (auto& e : edges) succ[f1[e.first]++] = e.second, pred[f2[e.second]++] = e.first;
  }
  std::vector<int> prio(T, 1);
  for (int64_t t = T - 1; t >= 0; --t)
    for (int64_t e = off[t]; e < off[t + 1]; ++e) prio[t] = std::max(prio[t], prio[succ[e]] + 1);
  auto is_diag = [&](int64_t t) { return ts[t] >= 0 && ts[t] == tb[t]; };
  double makespan = 0;
  {  // makespan estimate in steps: max(critical path, work / warps), tasks
     // weighted by their steps plus the fixed cost ovh
    std::vector<double> cp(T, 0.0);
    double work = 0, crit = 0;
    for (int64_t t = T - 1; t >= 0; --t) {
      const int wb = tb[t] == 0 ? W0 : W, wsg = ts[t] == 0 ? W0 : W;
      const double steps = (ts[t] < 0 ? 1.0 : is_diag(t) ? wb + 1.0 : double(wsg)) + ovh;
      work += steps * (is_diag(t) ? W / 2 : W) / 32.0;
      double best = 0;
      for (int64_t e = off[t]; e < off[t + 1]; ++e) best = std::max(best, cp[succ[e]]);
      cp[t] = steps + best;
      crit = std::max(crit, cp[t]);
    }
    makespan = std::max(crit, work / std::max<double>(1.0, procs * W / 32.0));
  }
  auto span = [&](int64_t t) { return is_diag(t) ? W / 16 : W / 8; };  // slots
  auto slot_of = [&](int64_t t) {
    const int j = tjob[t], b = tb[t], s2 = ts[t];
    if (s2 < 0) return make_int4(j, lo(b), 0, -3);
    if (s2 < b) return make_int4(j, lo(b), lo(s2), -1);
    return make_int4(j, lo(b), lo(b), -2);
  };

  // Packing into warp descriptors: a task goes to the earliest of the last
  // kOpen descriptors that has an aligned free position and follows all its
  // dependencies' descriptors, else to a new descriptor.
  BandSched out;
  out.makespan = makespan;
  std::vector<int> desc_of(T, -1);
  std::vector<std::array<int64_t, kSlots>> members;
  constexpr int kOpen = 64;
  std::vector<std::pair<int, unsigned>> openl;  // (descriptor, used-slot mask), ascending
  auto place = [&](std::vector<int4>& w, size_t wfirst, int64_t t) {
    const int sp = span(t);
    int latest = -1;
    for (int64_t e = poff[t]; e < poff[t + 1]; ++e) latest = std::max(latest, desc_of[pred[e]]);
    const int lim = static_cast<int>(members.size()) - kOpen;
    int dsc = -1, pos = -1;
    size_t oi = 0;
    for (; oi < openl.size(); ++oi) {
      const auto [q, used] = openl[oi];
      if (q <= latest || q < lim || q < static_cast<int>(wfirst)) continue;
      for (int f = 0; f + sp <= kSlots; f += sp)
        if (((used >> f) & ((1u << sp) - 1)) == 0) {
          dsc = q, pos = f;
          break;
        }
      if (dsc >= 0) break;
    }
    if (dsc < 0) {
      dsc = static_cast<int>(members.size());
      members.emplace_back();
      members.back().fill(-1);
      for (int f = 0; f < kSlots; ++f) w.push_back(make_int4(0, 0, 0, -4));
      openl.emplace_back(dsc, 0u);
      oi = openl.size() - 1;
      pos = 0;
    }
    const int4 v = slot_of(t);
    const size_t wb = (static_cast<size_t>(dsc) - wfirst) * kSlots;
    for (int f = pos; f < pos + sp; ++f) w[wb + f] = v;
    openl[oi].second |= ((1u << sp) - 1) << pos;
    members[dsc][pos] = t;
    desc_of[t] = dsc;
    if (openl[oi].second == (1u << kSlots) - 1) openl.erase(openl.begin() + static_cast<long>(oi));
    while (!openl.empty() && openl.front().first < static_cast<int>(members.size()) - kOpen) openl.erase(openl.begin());
  };

  if (flow) {
    // Greedy list scheduling simulated in time on `procs` task processors (a
    // task lasts its steps / W; a diagonal task, half the lanes, half that);
    // a task becomes ready `slack` after its last dependency finishes, so
    // in the resulting hand-out order a unit's dependencies are, where the
    // graph allows, a little more than one round of warps earlier.
    std::vector<int> indeg2 = indeg;
    std::vector<double> rt(T, 0.0);
    using Ev = std::pair<double, int64_t>;
    std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> pending;  // (ready time, task)
    std::priority_queue<std::pair<int, int64_t>> ready;                   // (prio, -task)
    std::priority_queue<double, std::vector<double>, std::greater<double>> procfree;
    for (int64_t q = 0; q < std::max<int64_t>(1, procs); ++q) procfree.push(0.0);
    for (int64_t t = 0; t < T; ++t)
      if (indeg2[t] == 0) pending.emplace(0.0, t);
    std::vector<int4> w;
    int64_t placed = 0;
    while (placed < T) {
      double now = procfree.top();
      while (!pending.empty() && pending.top().first <= now) {
        ready.emplace(prio[pending.top().second], -pending.top().second);
        pending.pop();
      }
      if (ready.empty()) {
        if (pending.empty()) throw std::logic_error("band schedule: dependency cycle");
        procfree.pop();
        procfree.push(pending.top().first);
        continue;
      }
      const int64_t t = -ready.top().second;
      ready.pop();
      procfree.pop();
      const int wb = tb[t] == 0 ? W0 : W, wsg = ts[t] == 0 ? W0 : W;
      const double dur = ts[t] < 0 ? 0.1 : is_diag(t) ? (wb + 1) / (2.0 * W) : double(wsg) / W;
      const double fin = now + dur;
      procfree.push(fin);
      place(w, 0, t);
      ++placed;
      for (int64_t e = off[t]; e < off[t + 1]; ++e) {
        const int64_t u = succ[e];
        rt[u] = std::max(rt[u], fin + slack);
        if (--indeg2[u] == 0) pending.emplace(rt[u], u);
      }
    }
    out.waves.push_back(std::move(w));
  } else {
    std::vector<int> indeg2 = indeg;
    std::priority_queue<std::pair<int, int64_t>> ready;  // (prio, -id)
    for (int64_t t = 0; t < T; ++t)
      if (indeg2[t] == 0) ready.emplace(prio[t], -t);
    int64_t done = 0;
    while (done < T) {
      if (ready.empty()) throw std::logic_error("band schedule: dependency cycle");
      std::vector<int64_t> picked;
      int64_t usedc = 0;
      while (!ready.empty() && usedc + span(-ready.top().second) <= std::max<int64_t>(cap_slots, kSlots)) {
        const int64_t t = -ready.top().second;
        ready.pop();
        usedc += span(t);
        picked.push_back(t);
      }
      // tasks of one wave are independent; pack the wide ones first
      std::stable_sort(picked.begin(), picked.end(), [&](int64_t x, int64_t y) { return span(x) > span(y); });
      std::vector<int4> w;
      const size_t wfirst = members.size();  // descriptors of earlier waves are closed
      for (int64_t t : picked) place(w, wfirst, t);
      out.waves.push_back(std::move(w));
      for (int64_t t : picked)
        for (int64_t e = off[t]; e < off[t + 1]; ++e)
          if (--indeg2[succ[e]] == 0) ready.emplace(prio[succ[e]], -succ[e]);
      done += static_cast<int64_t>(picked.size());
    }
  }
  // descriptor dependency lists
  out.dep_off.assign(1, 0);
  for (size_t dsc = 0; dsc < members.size(); ++dsc) {
    std::vector<int> ds;
    for (int64_t t : members[dsc]) {
      if (t < 0) continue;
      for (int64_t e = poff[t]; e < poff[t + 1]; ++e) {
        const int q = desc_of[pred[e]];
        if (q >= static_cast<int>(dsc)) throw std::logic_error("band schedule: dependency not scheduled earlier");
        ds.push_back(q);
      }
    }
    std::sort(ds.begin(), ds.end());
    ds.erase(std::unique(ds.begin(), ds.end()), ds.end());
    out.deps.insert(out.deps.end(), ds.begin(), ds.end());
    out.dep_off.push_back(static_cast<int>(out.deps.size()));
  }
  return out;
}

}  // namespace

struct Plan {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  int n = 0, N = 0, d = 0, m = 1, mode = 0, P = 1, Q = 1;
  int64_t TS = 0, TSdev = 0, top = 0;
  int max_batch = 1;
  Geom G{};
  const Launchers* L = nullptr;
  // Conv stage. Prologue layers (device exponent folding) run first on the
  // main stream; the graph's own conv jobs are partitioned into independent
  // groups (connected components of their dynamic slots, i.e. sets of whole
  // monomials) whose layer sequences run concurrently on their own streams.
  struct ConvGroup {
    std::vector<std::pair<int4*, int>> layers;  // (jobs, njobs) per layer
    std::vector<int> layer_index;                // graph conv layer of each entry
    cudaStream_t stream = nullptr;
    cudaEvent_t join = nullptr;
    double* prod = nullptr;  // split-path scratch of this group
    int64_t prod_words = 0;
  };
  std::vector<std::pair<int4*, int>> pro_layers;
  std::vector<ConvGroup> groups;
  cudaEvent_t fork = nullptr;
  std::vector<std::pair<int2*, int>> add_layers;  // non-empty graph add layers
  std::vector<int> add_layer_index;                // their graph add layer
  int n_conv_layers = 0, n_add_layers = 0;         // graph layers (RunReport entries)
  Stamp* stamps = nullptr;                         // phase stamps of the last run (device)
  std::vector<double> conv_layer_ms, add_layer_ms; // per-layer times of the last run
  double exchange_ms = 0;                          // sharded: conv end -> tail start
  // sharding one polynomial over devices: this plan's rank, and per rank the
  // dynamic slots the addition stage needs from that rank (device lists)
  int rank = 0, nranks = 1;
  std::vector<std::pair<int*, int>> xslots;
  std::vector<const double*> peer_arena;  // per rank (peer gather); opened IPC mappings are closed on destroy
  std::vector<bool> peer_ipc;
  // device copy of the peer list for the gather kernel, rebuilt when a peer changes
  PeerList* peer_list = nullptr;
  int64_t* peer_first = nullptr;
  int npeer_list = 0;
  int64_t peer_words1 = 0;  // words gathered per point
  bool peers_dirty = true;
  int2* ts = nullptr;
  int nts = 0;
  int* row_slot = nullptr;
  int* row_mult = nullptr;
  int nrows = 0;
  std::vector<void*> owned;
  // buffers
  double* arena = nullptr;
  double* stage = nullptr;  // [Q][max_batch][top][d+1]
  double* vg = nullptr;     // [Q][max_batch][n+1][d+1]
  double* dyn = nullptr;    // lazily: [Q][max_batch][TS][d+1]
  // split-convolution index table (k, i) of the triangular product index
  int2* tri = nullptr;
  int T = 0;
  int64_t split_threshold = 0;
  // accounting (per point)
  int64_t flops_model = 0, alg_ops = 0, conv_jobs = 0, add_jobs = 0, copy_jobs = 0;
  std::map<int, cudaGraphExec_t> graphs;
  std::vector<cudaEvent_t> ev;
  // Banded conv stage (see BandArgs): this rank's non-prologue conv jobs per
  // graph layer, and per batch size the banded part -- the conv layers from
  // `first` on, their job table and task schedule.
  std::vector<std::vector<ConvRow>> layer_rows;
  int64_t nrows_mine = 0;
  struct BandWaves {
    int first = 0;
    int W = 32;
    int4* jobs = nullptr;
    int4* tasks = nullptr;
    std::vector<std::pair<int64_t, int>> waves;  // (first descriptor, descriptors)
    int* dep_off = nullptr;  // flow mode
    int* deps = nullptr;
    unsigned* flags = nullptr;  // [batch][units]; per batch size, since a captured graph keeps its pointer
    int nunits = 0;
  };
  unsigned long long* flow_counter = nullptr;
  std::map<int, BandWaves> band_waves;
  int conv_mode = 0;         // PSE_CONV_MODE: 0 auto, 1 layered, 2 banded waves, 3 dataflow, 4 CTA-local dataflow
  double band_rounds = 1.0;  // PSE_BAND_ROUNDS: wave size in resident warps
  double flow_slack = 1.0;   // PSE_FLOW_SLACK: see band_schedule (swept: 0.1-8, best 1)
  int band_w = 0;            // PSE_BAND_W: 16 or 32 (0: chosen per run)
  double flow_procs = 1.0;   // PSE_FLOW_PROCS: simulated warps, as a fraction of the resident ones
  int64_t layer_pairs = 0;   // average conv layer size in coefficient pairs
  // some dynamic slot is written by more than one conv job (validate(), like
  // the reference, accepts a slot rewritten in a later layer): the banded
  // schedule assumes one producer per slot, so such graphs stay layered
  bool multi_writer = false;

  // First conv layer the banded path runs for this batch (layer_rows.size():
  // none). A layer is "small" when it offers less than two waves of resident
  // threads at one thread per coefficient pair. Deep graphs whose average
  // layer is small run banded throughout; otherwise the trailing run of small
  // layers (e.g. C2's last layer) runs banded after the layered ones.
  int band_first(int batch) const {
    const int nl = static_cast<int>(layer_rows.size());
    const int64_t nb16 = 1 + d / 16;  // bands at the narrow width: the schedule's size bound
    if (nrows_mine == 0 || conv_mode == 1 || multi_writer || nb16 > 32767 ||
        nrows_mine * nb16 * (nb16 + 1) / 2 >= (int64_t(1) << 31))
      return nl;
    if (conv_mode >= 2 || cta_mode()) return 0;  // waves, dataflow and CTA-local dataflow take every layer
    // Short chains (d < 24): a layer's critical path is short, so band tasks
    // have little to pipeline and add hand-out and flag costs -- layered wins
    // (conv stage, layered vs dataflow: C1 = p1 d=15 m=2 0.070 vs 0.117 ms;
    // p2 d=15 m=2 0.82 vs 1.40; p1 d=15 m=10 0.69 vs 0.92). At d=31 it is
    // mixed (p1 m=10 2.14 vs 1.54, p2 m=2 1.49 vs 1.85), at d=63 banded wins.
    if (d < 24) return nl;
    const int64_t thr = int64_t(sms) * 4 * 128 * 2, npairs = (d + 2) / 2;
    if (static_cast<int64_t>(batch) * layer_pairs < thr) return 0;
    int f = nl;
    while (f > 0 && static_cast<int64_t>(batch) * static_cast<int64_t>(layer_rows[f - 1].size()) * npairs < thr) --f;
    return f;
  }
  bool banded(int batch) const { return band_first(batch) < static_cast<int>(layer_rows.size()); }

  // the global dataflow kernel (also the CTA path's fallback)
  bool flow() const { return conv_mode == 3 || conv_mode == 0 || conv_mode == 4 || conv_mode == 5; }

  // ---- CTA-local dataflow (CtaArgs in kernels.cuh): one block per
  // independent job group (connected component of the dynamic slots: whole
  // monomials) and point; the group's banded tasks scheduled for one
  // block's warps. Built once (host only); ok = false when it cannot run
  // (a group's completion flags exceed shared memory next to the lanes).
  std::vector<std::vector<int>> layer_comp;  // component of every row of layer_rows
  int ncomps = 0;
  struct CtaPlan {
    bool built = false, ok = false;
    int W = 32, ngroups = 0, max_units = 0;
    int4 *jobs = nullptr, *tasks = nullptr;
    int *group_off = nullptr, *dep_off = nullptr, *deps = nullptr;
    double makespan = 0;  // simulated, in steps: the slowest group
    // layered form (k_conv_ctl): the group's layers in order, a block barrier
    // between them -- the M = 1 default (see prefer_cta) and PSE_CONV_MODE=ctl
    bool layered = false;
    int4* ljobs = nullptr;
    int *layer_off = nullptr, *lgroup_off = nullptr;
    int *stage_off = nullptr, *stage_slot = nullptr, *gjob_off = nullptr;  // see CtlArgs
    int4* sidx = nullptr;
    int max_stage = 0;
    size_t table_bytes = 0;
  } cta;

  // The CTA-local paths are taken when forced (PSE_CONV_MODE=cta: the band
  // tasks' dataflow, PSE_CONV_MODE=ctl: the layer walk) and, by default, for
  // every real graph at M = 1: the layer walk (k_conv_ctl) with the group's
  // operands in shared memory, whatever the group sizes -- C3 m=1 0.165 ms
  // conv (CTA-local dataflow 0.355, global dataflow 0.92), C2 m=1 0.091
  // (hybrid 0.30), C4 m=1 0.246 (layered 0.40), C1 m=1 0.031 (dataflow
  // 0.038). At M >= 2 the global kernels are faster (C3 m=2: dataflow 4.3 ms,
  // CTA-local dataflow 5.1, layer walk 8-17).
  bool prefer_cta() const {
    return conv_mode == 4 || conv_mode == 5 || (conv_mode == 0 && m == 1 && P == 1 && ncomps > 0);
  }
  bool cta_layered() const { return conv_mode == 5 || (conv_mode == 0 && m == 1); }
  bool cta_mode() const { return prefer_cta() && cta_ready(); }
  bool cta_ready() const { return cta.built && cta.ok; }

  void prepare_cta() {
    if (cta.built) return;
    cta.built = true;
    if (nrows_mine == 0 || multi_writer) return;
    const int64_t nb16 = 1 + d / 16;
    if (nb16 > 32767) return;
    // rows of each group, in layer order, and their layers
    std::vector<std::vector<ConvRow>> rows(ncomps);
    std::vector<std::vector<int>> rlayer(ncomps);
    for (size_t L2 = 0; L2 < layer_rows.size(); ++L2)
      for (size_t r = 0; r < layer_rows[L2].size(); ++r) {
        rows[layer_comp[L2][r]].push_back(layer_rows[L2][r]);
        rlayer[layer_comp[L2][r]].push_back(static_cast<int>(L2));
      }
    if (cta_layered()) {
      // jobs of each group layer by layer: (in1, in2, out, copy | layer << 8);
      // per (group, layer) the distinct input slots (M = 1 stages them in
      // shared memory), each job's staged (in1, in2) and the index of its
      // output in the next layer's list (-1: not read there)
      std::vector<int4> lj, si;
      std::vector<int> loff(1, 0), lgoff(1, 0), soff(1, 0), sslot, gjoff(1, 0);
      size_t table_bytes = 0;
      for (int c = 0; c < ncomps; ++c) {
        const size_t j_first = lj.size(), s_first = sslot.size(), l_first = loff.size() - 1;
        // layer boundaries of the group's rows
        std::vector<size_t> lb;
        for (size_t t = 0; t < rows[c].size(); ++t)
          if (t == 0 || rlayer[c][t] != rlayer[c][t - 1]) lb.push_back(t);
        lb.push_back(rows[c].size());
        std::vector<std::map<int64_t, int>> lists(lb.size() - 1);
        for (size_t q = 0; q + 1 < lb.size(); ++q) {
          std::map<int64_t, int>& st = lists[q];
          auto stage = [&](int64_t slot) {
            auto it = st.find(slot);
            if (it != st.end()) return it->second;
            const int e = static_cast<int>(st.size());
            st[slot] = e;
            return e;
          };
          std::set<int64_t> prev_out;
          if (q > 0)
            for (size_t t = lb[q - 1]; t < lb[q]; ++t) prev_out.insert(rows[c][t].out);
          std::vector<int64_t> order;
          for (size_t t = lb[q]; t < lb[q + 1]; ++t) {
            const ConvRow& r = rows[c][t];
            const size_t before = st.size();
            const int sx = stage(r.in1);
            if (st.size() > before) order.push_back(r.in1);
            int sy = sx;
            if (!r.copy) {
              const size_t b2 = st.size();
              sy = stage(r.in2);
              if (st.size() > b2) order.push_back(r.in2);
            }
            lj.push_back(make_int4(static_cast<int>(r.in1), static_cast<int>(r.in2), static_cast<int>(r.out),
                                   (r.copy ? 1 : 0) | (rlayer[c][t] << 8)));
            si.push_back(make_int4(sx, sy, -1, 0));
          }
          for (int64_t slot : order) sslot.push_back(static_cast<int>(slot * 2 + (prev_out.count(slot) ? 1 : 0)));
          loff.push_back(static_cast<int>(lj.size()));
          soff.push_back(static_cast<int>(sslot.size()));
          cta.max_stage = std::max(cta.max_stage, static_cast<int>(st.size()));
        }
        // outputs read by the next layer of the group
        for (size_t q = 0; q + 2 < lb.size(); ++q)
          for (size_t t = lb[q]; t < lb[q + 1]; ++t) {
            auto it = lists[q + 1].find(rows[c][t].out);
            if (it != lists[q + 1].end()) si[j_first + t].z = it->second;
          }
        lgoff.push_back(static_cast<int>(loff.size()) - 1);
        gjoff.push_back(static_cast<int>(lj.size()));
        const size_t nj = lj.size() - j_first, nl = loff.size() - 1 - l_first, ns = sslot.size() - s_first;
        table_bytes = std::max(table_bytes, nj * 2 * sizeof(int4) + 2 * (nl + 1) * sizeof(int) + ns * sizeof(int));
      }
      if (!L->ctl_fits(cta.max_stage, d, table_bytes)) return;  // stays on the global dataflow path
      cta.table_bytes = table_bytes;
      cta.ngroups = ncomps;
      cta.ljobs = dev_upload(lj, stream);
      cta.layer_off = dev_upload(loff, stream);
      cta.lgroup_off = dev_upload(lgoff, stream);
      cta.stage_off = dev_upload(soff, stream);
      cta.stage_slot = dev_upload(sslot.empty() ? std::vector<int>{0} : sslot, stream);
      cta.sidx = dev_upload(si, stream);
      cta.gjob_off = dev_upload(gjoff, stream);
      ck(cudaStreamSynchronize(stream), "ctl upload");
      cta.layered = true;
      cta.ok = true;
      return;
    }
    const int warps = L->threads / 32;
    const Costs cst = costs(m);
    // fixed cost of a task (shared-memory hand-out and flags) in steps
    const double ovh = 250.0 / static_cast<double>(cst.inst_mul + cst.inst_add);
    std::vector<int4> jobs, tasks;
    std::vector<int> goff(1, 0), doff(1, 0), deps;
    for (int c = 0; c < ncomps; ++c)  // a group too large to schedule stays on the global path
      if (static_cast<int64_t>(rows[c].size()) * nb16 * (nb16 + 1) / 2 >= (int64_t(1) << 31)) return;
    auto sched_all = [&](int W) {
      double worst = 0;
      for (int c = 0; c < ncomps; ++c) {
        if (rows[c].empty()) continue;
        const BandSched sc = band_schedule(rows[c], d, W, kSlots, true, int64_t(warps) * (32 / W), flow_slack, ovh);
        worst = std::max(worst, sc.makespan);
        const int jbase = static_cast<int>(jobs.size());
        std::set<int64_t> produced;
        for (auto& r : rows[c]) produced.insert(r.out);
        for (size_t t = 0; t < rows[c].size(); ++t) {
          const ConvRow& r = rows[c][t];
          jobs.push_back(make_int4(static_cast<int>(r.in1), static_cast<int>(r.in2), static_cast<int>(r.out),
                                   (produced.count(r.in1) ? 2 : 0) | (!r.copy && produced.count(r.in2) ? 4 : 0) |
                                       (rlayer[c][t] << 8)));
        }
        const std::vector<int4>& w = sc.waves.at(0);
        for (int4 v : w) {
          if (v.w != -4) v.x += jbase;
          tasks.push_back(v);
        }
        const int nd = static_cast<int>(w.size() / kSlots);
        cta.max_units = std::max(cta.max_units, nd);
        for (int q = 0; q < nd; ++q) {
          for (int e = sc.dep_off[q]; e < sc.dep_off[q + 1]; ++e) deps.push_back(sc.deps[e]);
          doff.push_back(static_cast<int>(deps.size()));
        }
        goff.push_back(goff.back() + nd);
      }
      return worst;
    };
    // 32-wide bands: a block's warps are few, so fewer, longer tasks win
    // (C3 m=1: 0.39 ms at W=32 vs 0.78 at 16); PSE_BAND_W overrides
    cta.W = band_w ? band_w : 32;
    cta.makespan = sched_all(cta.W);
    cta.ngroups = static_cast<int>(goff.size()) - 1;
    if (!L->cta_fits(cta.max_units)) return;  // stays on the global dataflow path
    cta.jobs = dev_upload(jobs, stream);
    cta.tasks = dev_upload(tasks, stream);
    cta.group_off = dev_upload(goff, stream);
    cta.dep_off = dev_upload(doff, stream);
    cta.deps = dev_upload(deps.empty() ? std::vector<int>{0} : deps, stream);
    ck(cudaStreamSynchronize(stream), "cta upload");
    cta.ok = true;
  }

  // host schedule + upload for a batch size (never during stream capture)
  void prepare_band(int batch) {
    if (prefer_cta()) {
      prepare_cta();
      if (cta_ready()) return;
    }
    if (!banded(batch) || band_waves.count(batch)) return;
    BandWaves bw;
    bw.first = band_first(batch);
    std::vector<ConvRow> rows;
    std::vector<int> row_layer;
    for (size_t L2 = bw.first; L2 < layer_rows.size(); ++L2) {
      rows.insert(rows.end(), layer_rows[L2].begin(), layer_rows[L2].end());
      row_layer.insert(row_layer.end(), layer_rows[L2].size(), static_cast<int>(L2));
    }
    {  // job table; flag bits 2/4: in1/in2 produced inside the banded part;
       // bits 8+: the graph conv layer (phase stamps)
      std::set<int64_t> produced;
      for (auto& r : rows) produced.insert(r.out);
      std::vector<int4> v;
      for (size_t t = 0; t < rows.size(); ++t) {
        const ConvRow& r = rows[t];
        v.push_back(make_int4(static_cast<int>(r.in1), static_cast<int>(r.in2), static_cast<int>(r.out),
                              (produced.count(r.in1) ? 2 : 0) | (!r.copy && produced.count(r.in2) ? 4 : 0) |
                                  (row_layer[t] << 8)));
      }
      bw.jobs = dev_upload(v, stream);
    }
    const int warps = sms * L->band_blocks_per_sm(flow()) * (L->threads / 32);
    const int64_t cap_slots = std::max<int64_t>(kSlots, static_cast<int64_t>(kSlots * band_rounds * warps / batch));
    // per-task fixed cost in steps: ~4 us of hand-out / flags / partial sums
    // against one md_mul + md_add (instrumented ops; ~2000 ops per us-warp)
    const Costs cst = costs(m);
    const double ovh = 2000.0 / static_cast<double>(cst.inst_mul + cst.inst_add);
    auto sched = [&](int W) {
      const int64_t procs = std::max<int64_t>(1, static_cast<int64_t>(flow_procs * warps / batch)) * (32 / W);
      return band_schedule(rows, d, W, cap_slots, flow(), procs, flow_slack, ovh);
    };
    // Band width: 16 halves the dependency chain of a deep graph (dataflow
    // critical path), 32 halves the number of tasks; in flow mode the one
    // with the shorter simulated makespan wins unless PSE_BAND_W fixes it.
    BandSched sch;
    if (band_w || !flow()) {
      bw.W = band_w ? band_w : 32;
      sch = sched(bw.W);
    } else {
      BandSched s16 = sched(16), s32 = sched(32);
      const bool narrow = s16.makespan < s32.makespan;
      bw.W = narrow ? 16 : 32;
      sch = std::move(narrow ? s16 : s32);
    }
    std::vector<int4> all;
    for (auto& w : sch.waves) {
      bw.waves.emplace_back(static_cast<int64_t>(all.size() / kSlots), static_cast<int>(w.size() / kSlots));
      all.insert(all.end(), w.begin(), w.end());
    }
    bw.tasks = dev_upload(all, stream);
    bw.nunits = static_cast<int>(all.size() / kSlots);
    if (flow()) {
      bw.dep_off = dev_upload(sch.dep_off, stream);
      bw.deps = dev_upload(sch.deps, stream);
      bw.flags = dev_alloc<unsigned>(static_cast<size_t>(batch) * bw.nunits);
      if (!flow_counter) flow_counter = dev_alloc<unsigned long long>(1);
    }
    ck(cudaStreamSynchronize(stream), "band upload");
    band_waves.emplace(batch, std::move(bw));
  }

  ~Plan() {
    if (device >= 0) cudaSetDevice(device);
    for (auto& [b, g] : graphs) cudaGraphExecDestroy(g);
    for (auto& [b, w] : band_waves) {
      cudaFree(w.tasks);
      cudaFree(w.jobs);
      cudaFree(w.dep_off);
      cudaFree(w.deps);
      cudaFree(w.flags);
    }
    cudaFree(flow_counter);
    cudaFree(cta.jobs);
    cudaFree(cta.tasks);
    cudaFree(cta.group_off);
    cudaFree(cta.dep_off);
    cudaFree(cta.deps);
    cudaFree(cta.ljobs);
    cudaFree(cta.layer_off);
    cudaFree(cta.lgroup_off);
    cudaFree(cta.stage_off);
    cudaFree(cta.stage_slot);
    cudaFree(cta.sidx);
    cudaFree(cta.gjob_off);
    cudaFree(stamps);
    cudaFree(peer_list);
    cudaFree(peer_first);
    for (cudaEvent_t x : ev) cudaEventDestroy(x);
    for (void* p : owned) cudaFree(p);
    cudaFree(arena);
    cudaFree(stage);
    cudaFree(vg);
    cudaFree(dyn);
    cudaFree(tri);
    for (size_t r = 0; r < peer_arena.size(); ++r)
      if (peer_ipc[r] && peer_arena[r]) cudaIpcCloseMemHandle(const_cast<double*>(peer_arena[r]));
    for (ConvGroup& gr : groups) {
      cudaFree(gr.prod);
      if (gr.join) cudaEventDestroy(gr.join);
      if (gr.stream) cudaStreamDestroy(gr.stream);
    }
    if (fork) cudaEventDestroy(fork);
    if (stream) cudaStreamDestroy(stream);
  }

  // launch the whole phase sequence; if ts is non-null, record an event
  // after every phase into ts (conv layers, scale, add layers, extract)
  // A conv layer runs split (products in parallel, then the accumulation
  // chains) when one thread per coefficient pair cannot fill the GPU.
  // The threshold is per group: concurrent groups share the GPU.
  bool split_layer(int nj, int batch, const ConvGroup& gr) const {
    return gr.prod != nullptr &&
           static_cast<int64_t>(batch) * nj * ((d + 2) / 2) * static_cast<int64_t>(groups.size()) < split_threshold &&
           static_cast<int64_t>(batch) * nj * T * Q <= gr.prod_words;
  }

  // ---- phase stamps (see Stamp in kernels.cuh): [0] conv start, [1 + L] end
  // of graph conv layer L, then the tail's start, the scale end, the add
  // layer ends and the extract end. Start slots hold inverted times.
  Stamp* stamp_conv(int layer) const { return layer < 0 ? nullptr : stamps + 1 + layer; }
  Stamp* stamp_tail_begin() const { return stamps + 1 + n_conv_layers; }
  Stamp* stamp_scale() const { return stamps + 2 + n_conv_layers; }
  Stamp* stamp_add(int layer) const { return stamps + 3 + n_conv_layers + layer; }
  Stamp* stamp_extract() const { return stamps + 3 + n_conv_layers + n_add_layers; }
  int nstamps() const { return 4 + n_conv_layers + n_add_layers; }

  // layer: graph conv layer (-1 = a prologue fold layer, not stamped)
  int launch_layer(int4* jobs, int nj, int batch, const ConvGroup& gr, cudaStream_t st, int layer) {
    Stamp* b = layer < 0 ? nullptr : stamps;
    if (split_layer(nj, batch, gr)) {
      SplitArgs a{arena, G, jobs, nj, batch, gr.prod, tri, T, b, stamp_conv(layer)};
      L->conv_prod(a, st);
      L->conv_accum(a, st);
      return 2;
    }
    ConvArgs a{arena, G, jobs, nj, (d + 2) / 2, batch, b, stamp_conv(layer)};
    L->conv(a, st);
    return 1;
  }

  // whole evaluation; a sharded plan (nranks > 1) runs only its conv share
  // here and the tail after the exchange (pse_plan_finish)
  int launch_all(int batch) {
    const int n = launch_conv(batch);
    return nranks > 1 ? n : n + launch_tail(batch);
  }

  int launch_conv(int batch) {
    int launches = 0;
    ck(cudaMemsetAsync(stamps, 0, sizeof(Stamp) * nstamps(), stream), "stamps");
    for (auto& [jobs, nj] : pro_layers) launches += launch_layer(jobs, nj, batch, groups[0], stream, -1);
    const int first = band_first(batch);
    if (first > 0) {  // layered part: graph conv layers < first
      if (groups.size() == 1) {
        for (size_t q = 0; q < groups[0].layers.size(); ++q) {
          const int li = groups[0].layer_index[q];
          if (li >= first) continue;
          launches += launch_layer(groups[0].layers[q].first, groups[0].layers[q].second, batch, groups[0], stream, li);
        }
      } else {
        ck(cudaEventRecord(fork, stream), "fork");
        for (ConvGroup& gr : groups) {
          ck(cudaStreamWaitEvent(gr.stream, fork, 0), "fork wait");
          for (size_t q = 0; q < gr.layers.size(); ++q)
            if (gr.layer_index[q] < first)
              launches += launch_layer(gr.layers[q].first, gr.layers[q].second, batch, gr, gr.stream, gr.layer_index[q]);
          ck(cudaEventRecord(gr.join, gr.stream), "join");
          ck(cudaStreamWaitEvent(stream, gr.join, 0), "join wait");
        }
      }
    }
    if (first < static_cast<int>(layer_rows.size()) && cta_mode() && cta.layered) {  // CTA-local layers
      CtlArgs a{arena,         G,          cta.ljobs, cta.layer_off,  cta.lgroup_off, cta.ngroups, batch, (d + 2) / 2,
                stamps,        cta.stage_off, cta.stage_slot, cta.sidx, cta.gjob_off, cta.max_stage};
      L->conv_ctl(a, cta.table_bytes, stream);
      ++launches;
    } else if (first < static_cast<int>(layer_rows.size()) && cta_mode()) {  // CTA-local dataflow
      CtaArgs a{arena, G, cta.jobs, cta.tasks, cta.group_off, cta.dep_off, cta.deps, cta.ngroups, batch, cta.W, stamps};
      if (!L->conv_cta(a, cta.max_units, stream)) throw std::logic_error("CTA-local dataflow does not fit");
      ++launches;
    } else if (first < static_cast<int>(layer_rows.size())) {  // banded part
      const BandWaves& bw = band_waves.at(batch);
      if (flow()) {
        ck(cudaMemsetAsync(bw.flags, 0, sizeof(unsigned) * batch * bw.nunits, stream), "flags");
        ck(cudaMemsetAsync(flow_counter, 0, sizeof(unsigned long long), stream), "counter");
        FlowArgs a{arena, G, bw.jobs, bw.tasks, bw.dep_off, bw.deps, bw.nunits, batch, bw.flags, flow_counter, bw.W, stamps};
        L->conv_flow(a, sms * L->band_blocks_per_sm(true), stream);
        ++launches;
      } else {
        for (auto& [o, nw] : bw.waves) {
          BandArgs a{arena, G, bw.jobs, bw.tasks + o * kSlots, nw, batch, bw.W, stamps};
          L->conv_band(a, stream);
          ++launches;
        }
      }
    }
    return launches;
  }

  // term scales, addition layers, extraction
  int launch_tail(int batch) {
    int launches = 0;
    Stamp* tb = stamp_tail_begin();
    if (nts) {
      ScaleArgs a{arena, G, ts, nts, batch, tb, stamp_scale()};
      L->scale(a, stream);
      ++launches;
    }
    for (size_t q = 0; q < add_layers.size(); ++q) {
      AddArgs a{arena, G, add_layers[q].first, add_layers[q].second, batch, tb, stamp_add(add_layer_index[q])};
      L->add(a, stream);
      ++launches;
    }
    ExtractArgs e{arena, G, row_slot, row_mult, nrows, batch, vg, tb, stamp_extract()};
    L->extract(e, stream);
    ++launches;
    return launches;
  }

  // Phase times of the last run from the stamps (synchronous D2H of a few
  // words). A phase ends when every job of it AND of the earlier phases is
  // done (layers of independent monomials overlap on the device), so the
  // per-layer times are non-negative and add up to the stage times. The
  // reference's wall_ms covers the conv, scale and add phases
  // (executor.cpp:168-183); the extraction is outside it, as there.
  void read_stamps(pse_report* rep, bool tail) {
    std::vector<Stamp> h(nstamps());
    ck(cudaMemcpyAsync(h.data(), stamps, sizeof(Stamp) * h.size(), cudaMemcpyDeviceToHost, stream), "stamps D2H");
    ck(cudaStreamSynchronize(stream), "stamps");
    auto ms = [](Stamp a, Stamp b) { return b > a ? static_cast<double>(b - a) * 1e-6 : 0.0; };
    const Stamp t0 = ~h[0];  // 0 (no conv kernel ran) -> ~0
    Stamp at = h[0] ? t0 : 0;
    conv_layer_ms.assign(n_conv_layers, 0.0);
    for (int l = 0; l < n_conv_layers; ++l) {
      const Stamp e = std::max(at, h[1 + l]);
      conv_layer_ms[l] = at ? ms(at, e) : 0.0;
      at = e;
    }
    Stamp conv_end = at;
    add_layer_ms.assign(n_add_layers, 0.0);
    double scale = 0, add = 0;
    Stamp tail_end = conv_end;
    if (tail) {
      // a sharded plan's tail starts after the exchange (barriers + gather);
      // otherwise the launch gap belongs to the first tail phase. A rank
      // without conv jobs (more ranks than job groups) has no conv stage:
      // its evaluation starts with the tail.
      const Stamp tb = h[1 + n_conv_layers] ? ~h[1 + n_conv_layers] : conv_end;
      if (!h[0]) conv_end = tb;
      at = nranks > 1 ? std::max(tb, conv_end) : conv_end;
      exchange_ms = nranks > 1 ? ms(conv_end, at) : 0.0;
      if (nts) {
        const Stamp e = std::max(at, h[2 + n_conv_layers]);
        scale = ms(at, e);
        at = e;
      }
      for (int l = 0; l < n_add_layers; ++l) {
        const Stamp e = std::max(at, h[3 + n_conv_layers + l]);
        add_layer_ms[l] = ms(at, e);
        add += add_layer_ms[l];
        at = e;
      }
      tail_end = at;
    }
    if (rep) {
      double conv = 0;
      for (double x : conv_layer_ms) conv += x;
      rep->conv_ms = conv;
      rep->scale_ms = scale;
      rep->add_ms = add;
      rep->wall_ms = h[0] ? ms(t0, tail_end) : exchange_ms + scale + add;
    }
  }

  void ensure_events(int k) {
    while (static_cast<int>(ev.size()) < k) {
      cudaEvent_t x;
      ck(cudaEventCreate(&x), "event create");
      ev.push_back(x);
    }
  }

  int kernel_count(int batch) const {
    int n = nranks > 1 ? 0 : (nts ? 1 : 0) + static_cast<int>(add_layers.size()) + 1;
    for (auto& [jobs, nj] : pro_layers) n += split_layer(nj, batch, groups[0]) ? 2 : 1;
    const int first = band_first(batch);
    if (first < static_cast<int>(layer_rows.size()))
      n += cta_mode() || flow() ? 1 : static_cast<int>(band_waves.at(batch).waves.size());
    for (const ConvGroup& gr : groups)
      for (size_t q = 0; q < gr.layers.size(); ++q)
        if (gr.layer_index[q] < first) n += split_layer(gr.layers[q].second, batch, gr) ? 2 : 1;
    return n;
  }
};

namespace {

// Build the device plan: validate, version in-place slots, add optional
// prologue (fold) jobs, upload job tables, allocate the arena.
Plan* build_plan(const pse_graph_desc& g, int device, int max_batch, const std::vector<std::vector<ConvRow>>& prologue,
                 int64_t prologue_slots, int rank = 0, int nranks = 1) {
  if (!valid_precision(g.m)) throw std::invalid_argument("unsupported precision level");
  if (g.mode != PSE_MODE_REAL && g.mode != PSE_MODE_COMPLEX) throw std::invalid_argument("unsupported mode");
  if (max_batch < 1) throw std::invalid_argument("max_batch must be at least 1");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / rank count");
  const std::string why = validate_desc(g);
  if (!why.empty()) throw std::invalid_argument("invalid job graph: " + why);
  if (g.total_slots + prologue_slots + g.conv_layer_off[g.n_conv_layers] >= (int64_t(1) << 31))
    throw std::invalid_argument("graph too large for 32-bit slot indices");

  std::unique_ptr<Plan> p(new Plan);
  p->device = device;
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device), "attr");
  ck(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "stream");
  p->n = g.n;
  p->N = g.N;
  p->d = g.d;
  p->m = g.m;
  p->mode = g.mode;
  p->P = g.mode == PSE_MODE_COMPLEX ? 2 : 1;
  p->Q = p->P * g.m;
  p->TS = g.total_slots;
  p->top = 1 + static_cast<int64_t>(g.N) + g.n;
  p->max_batch = max_batch;
  p->rank = rank;
  p->nranks = nranks;
  p->L = launchers_for(g.m, g.mode == PSE_MODE_COMPLEX);
  p->L->prepare();

  // conv rows per layer: prologue layers first, then the graph's layers
  int64_t next_slot = g.total_slots + prologue_slots;
  std::vector<std::vector<ConvRow>> layers = versioned_layers(g, prologue, &next_slot);
  for (int64_t t = 0; t < g.conv_layer_off[g.n_conv_layers]; ++t) p->copy_jobs += g.conv_copy[t] ? 1 : 0;
  p->TSdev = next_slot;
  p->G.d = g.d;
  p->G.S = (g.d + 1 + 3) / 4 * 4;
  p->G.Q = p->Q;
  p->G.slot_words = static_cast<int64_t>(p->Q) * p->G.S;
  p->G.point_words = p->TSdev * p->G.slot_words;

  cudaStream_t s = p->stream;
  auto upload_rows = [&](const std::vector<ConvRow>& rows) {
    std::vector<int4> v;
    v.reserve(rows.size());
    for (auto& r : rows)
      v.push_back(make_int4(static_cast<int>(r.in1), static_cast<int>(r.in2), static_cast<int>(r.out), r.copy));
    int4* dv = dev_upload(v, s);
    p->owned.push_back(dv);
    return std::make_pair(dv, static_cast<int>(v.size()));
  };
  const size_t npro = prologue.size();
  for (size_t L = 0; L < npro; ++L)
    if (!layers[L].empty()) p->pro_layers.push_back(upload_rows(layers[L]));

  // Independent job groups: union-find over dynamic slots (>= top) of every
  // non-prologue conv job; components (whole monomials) are dealt out in
  // contiguous ranges of first appearance, balanced by job count.
  {
    std::map<int64_t, int64_t> parent;
    std::function<int64_t(int64_t)> find = [&](int64_t x) {
      auto it = parent.find(x);
      if (it == parent.end()) {
        parent[x] = x;
        return x;
      }
      if (it->second == x) return x;
      const int64_t r = find(it->second);
      parent[x] = r;
      return r;
    };
    auto unite = [&](int64_t a, int64_t b) {
      a = find(a);
      b = find(b);
      if (a != b) parent[a] = b;
    };
    const int64_t top = p->top;
    int64_t njobs = 0;
    for (size_t L = npro; L < layers.size(); ++L)
      for (const ConvRow& r : layers[L]) {
        find(r.out);
        if (r.in1 >= top) unite(r.in1, r.out);
        if (!r.copy && r.in2 >= top) unite(r.in2, r.out);
        ++njobs;
      }
    std::map<int64_t, int64_t> comp_jobs;  // root -> jobs
    std::vector<int64_t> comp_order;
    for (size_t L = npro; L < layers.size(); ++L)
      for (const ConvRow& r : layers[L]) {
        const int64_t c = find(r.out);
        if (!comp_jobs.count(c)) comp_order.push_back(c);
        ++comp_jobs[c];
      }
    // Sharding one polynomial over `nranks` devices: components are dealt to
    // ranks in contiguous ranges balanced by job count; this plan keeps only
    // its rank's jobs (then split into concurrent groups as usual).
    std::map<int64_t, int> comp_rank;
    {
      int64_t acc = 0;
      for (int64_t c : comp_order) {
        comp_rank[c] = static_cast<int>(std::min<int64_t>(nranks - 1, acc * nranks / std::max<int64_t>(1, njobs)));
        acc += comp_jobs[c];
      }
    }
    std::vector<int64_t> mine;
    int64_t njobs_mine = 0;
    for (int64_t c : comp_order)
      if (comp_rank[c] == rank) {
        mine.push_back(c);
        njobs_mine += comp_jobs[c];
      }
    const char* env = getenv("PSE_CONV_GROUPS");
    int ng = env ? atoi(env) : 4;
    ng = std::max(1, std::min<int>(ng, static_cast<int>(mine.size())));
    std::map<int64_t, int> comp_group, comp_index;
    for (int64_t c : mine) comp_index[c] = static_cast<int>(comp_index.size());
    p->ncomps = static_cast<int>(mine.size());
    int64_t acc = 0;
    for (int64_t c : mine) {
      comp_group[c] = static_cast<int>(std::min<int64_t>(ng - 1, acc * ng / std::max<int64_t>(1, njobs_mine)));
      acc += comp_jobs[c];
    }
    p->groups.resize(ng);
    int64_t nlayers = 0;
    for (size_t L = npro; L < layers.size(); ++L) {
      std::vector<std::vector<ConvRow>> per(ng);
      p->layer_rows.emplace_back();
      p->layer_comp.emplace_back();
      for (const ConvRow& r : layers[L]) {
        const int64_t root = find(r.out);
        auto it = comp_group.find(root);
        if (it != comp_group.end()) {
          per[it->second].push_back(r);
          p->layer_rows.back().push_back(r);
          p->layer_comp.back().push_back(comp_index[root]);
          ++p->nrows_mine;
        }
      }
      if (!layers[L].empty()) ++nlayers;
      for (int gi = 0; gi < ng; ++gi)
        if (!per[gi].empty()) {
          p->groups[gi].layers.push_back(upload_rows(per[gi]));
          p->groups[gi].layer_index.push_back(static_cast<int>(L - npro));
        }
    }
    p->layer_pairs = p->nrows_mine * ((g.d + 2) / 2) / std::max<int64_t>(1, nlayers);
    {
      std::set<int64_t> outs;
      for (const auto& lr : p->layer_rows)
        for (const ConvRow& r : lr)
          if (!outs.insert(r.out).second) p->multi_writer = true;
    }
    {
      const char* cm = getenv("PSE_CONV_MODE");
      const std::string m = cm ? cm : "";
      p->conv_mode = m == "layer" ? 1 : m == "band" ? 2 : m == "flow" ? 3 : m == "cta" ? 4 : m == "ctl" ? 5 : 0;
      const char* br = getenv("PSE_BAND_ROUNDS");
      if (br && atof(br) > 0) p->band_rounds = atof(br);
      const char* fs = getenv("PSE_FLOW_SLACK");
      if (fs && atof(fs) >= 0) p->flow_slack = atof(fs);
      const char* fp = getenv("PSE_FLOW_PROCS");
      if (fp && atof(fp) > 0) p->flow_procs = atof(fp);
      const char* bwv = getenv("PSE_BAND_W");
      if (bwv && (atoi(bwv) == 16 || atoi(bwv) == 32)) p->band_w = atoi(bwv);
    }
    // exchange lists: every dynamic slot the addition stage, the term scales
    // or the extraction reads, by the rank whose conv jobs produce it
    if (nranks > 1) {
      std::set<int64_t> need;
      for (int64_t t = 0; t < g.add_layer_off[g.n_add_layers]; ++t) {
        need.insert(g.add_src[t]);
        need.insert(g.add_dst[t]);
      }
      for (int64_t t = 0; t < g.n_term_scales; ++t) need.insert(g.ts_slot[t]);
      need.insert(g.value_slot);
      for (int i = 0; i < g.n; ++i)
        if (g.gradient_slots[i] >= 0) need.insert(g.gradient_slots[i]);
      std::vector<std::vector<int>> lists(nranks);
      for (int64_t s : need)
        if (s >= top) lists[comp_rank[find(s)]].push_back(static_cast<int>(s));
      p->xslots.resize(nranks);
      for (int r2 = 0; r2 < nranks; ++r2) {
        p->xslots[r2].second = static_cast<int>(lists[r2].size());
        p->xslots[r2].first = lists[r2].empty() ? nullptr : dev_upload(lists[r2], s);
        if (p->xslots[r2].first) p->owned.push_back(p->xslots[r2].first);
      }
    }
    if (ng > 1) {
      ck(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming), "event");
      for (auto& gr : p->groups) {
        ck(cudaStreamCreateWithFlags(&gr.stream, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreateWithFlags(&gr.join, cudaEventDisableTiming), "event");
      }
    }
  }
  for (int32_t L = 0; L < g.n_add_layers; ++L) {
    std::vector<int2> v;
    for (int64_t t = g.add_layer_off[L]; t < g.add_layer_off[L + 1]; ++t)
      v.push_back(make_int2(static_cast<int>(g.add_src[t]), static_cast<int>(g.add_dst[t])));
    if (v.empty()) continue;
    int2* dv = dev_upload(v, s);
    p->owned.push_back(dv);
    p->add_layers.emplace_back(dv, static_cast<int>(v.size()));
    p->add_layer_index.push_back(L);
  }
  p->n_conv_layers = g.n_conv_layers;
  p->n_add_layers = g.n_add_layers;
  p->stamps = dev_alloc<Stamp>(static_cast<size_t>(p->nstamps()));
  if (g.n_term_scales) {
    std::vector<int2> v;
    for (int64_t t = 0; t < g.n_term_scales; ++t) {
      if (g.ts_factor[t] > (int64_t(1) << 30) || g.ts_factor[t] < -(int64_t(1) << 30))
        throw std::invalid_argument("term scale factor out of range");
      v.push_back(make_int2(static_cast<int>(g.ts_slot[t]), static_cast<int>(g.ts_factor[t])));
    }
    p->ts = dev_upload(v, s);
    p->owned.push_back(p->ts);
    p->nts = static_cast<int>(v.size());
  }
  std::vector<int> rs(g.n + 1), rm(g.n + 1, 1);
  rs[0] = static_cast<int>(g.value_slot);
  for (int i = 0; i < g.n; ++i) {
    rs[1 + i] = g.gradient_slots[i] < 0 ? -1 : static_cast<int>(g.gradient_slots[i]);
    if (g.multipliers[i] > (int64_t(1) << 30) || g.multipliers[i] < -(int64_t(1) << 30))
      throw std::invalid_argument("multiplier out of range");
    rm[1 + i] = static_cast<int>(g.multipliers[i]);
  }
  p->nrows = g.n + 1;
  p->row_slot = dev_upload(rs, s);
  p->row_mult = dev_upload(rm, s);
  p->owned.push_back(p->row_slot);
  p->owned.push_back(p->row_mult);

  // Split-convolution scratch: sized for the largest (batch x layer) that
  // the threshold sends down the split path, capped at 4 GiB (layers beyond
  // the cap simply stay fused). Threshold: two waves of resident threads
  // (4 blocks of 128 per SM); PSE_SPLIT_THRESHOLD overrides, 0 disables.
  {
    const char* env = getenv("PSE_SPLIT_THRESHOLD");
    p->split_threshold = env ? atoll(env) : int64_t(p->sms) * 4 * 128 * 2;
    p->T = (g.d + 1) * (g.d + 2) / 2;
    const int64_t npairs = (g.d + 2) / 2, ng = static_cast<int64_t>(p->groups.size());
    auto words_for = [&](const std::vector<std::pair<int4*, int>>& ls) {
      int64_t need = 0;
      for (auto& [jobs, nj] : ls) {
        int64_t bmax = 0;
        for (int b = max_batch; b >= 1; --b)
          if (int64_t(b) * nj * npairs * ng < p->split_threshold) {
            bmax = b;
            break;
          }
        need = std::max(need, bmax * nj * int64_t(p->T) * p->Q);
      }
      return std::min<int64_t>(need, (int64_t(4) << 30) / 8 / ng);
    };
    bool any = false;
    for (size_t gi = 0; gi < p->groups.size(); ++gi) {
      Plan::ConvGroup& gr = p->groups[gi];
      int64_t need = words_for(gr.layers);
      if (gi == 0) need = std::max(need, words_for(p->pro_layers));
      if (need > 0) {
        gr.prod = dev_alloc<double>(static_cast<size_t>(need));
        gr.prod_words = need;
        any = true;
      }
    }
    if (any) {
      std::vector<int2> tri(p->T);
      for (int k = 0, o = 0; k <= g.d; ++k)
        for (int i = 0; i <= k; ++i) tri[o++] = make_int2(k, i);
      p->tri = dev_upload(tri, s);
    }
  }

  p->arena = dev_alloc<double>(static_cast<size_t>(max_batch) * p->G.point_words);
  p->stage = dev_alloc<double>(static_cast<size_t>(p->Q) * max_batch * p->top * (g.d + 1));
  p->vg = dev_alloc<double>(static_cast<size_t>(p->Q) * max_batch * p->nrows * (g.d + 1));
  ck(cudaStreamSynchronize(s), "plan upload");

  if (p->prefer_cta()) p->prepare_cta();
  const Costs c = costs(g.m);
  p->flops_model = flop_count(g, 0, c.rep_add, c.rep_mul);
  p->alg_ops = alg_op_count(g);
  p->conv_jobs = g.conv_layer_off[g.n_conv_layers];
  p->add_jobs = g.add_layer_off[g.n_add_layers];
  return p.release();
}

void fill_report(const Plan& p, int batch, pse_report* rep) {
  rep->double_op_count = p.flops_model;
  rep->alg_op_count = p.alg_ops;
  rep->conv_jobs_executed = p.conv_jobs * batch;
  rep->add_jobs_executed = p.add_jobs * batch;
  rep->copy_jobs_executed = p.copy_jobs * batch;
  rep->batch = batch;
}

void upload(Plan& p, int batch, const double* const* slabs, int64_t stride) {
  if (batch < 1 || batch > p.max_batch) throw std::invalid_argument("batch outside [1, max_batch]");
  if (!slabs) throw std::invalid_argument("null static slabs");
  const int64_t pw = p.top * (p.d + 1);
  if (stride == 0) stride = pw;
  if (stride < pw) throw std::invalid_argument("point stride smaller than the static region");
  ck(cudaSetDevice(p.device), "cudaSetDevice");
  // slabs may be host (pinned or pageable) or device pointers (UVA decides):
  // device-resident inputs are staged with a D2D copy
  for (int q = 0; q < p.Q; ++q) {
    if (!slabs[q]) throw std::invalid_argument("null static slab");
    double* dst = p.stage + static_cast<int64_t>(q) * batch * pw;
    if (stride == pw) {
      ck(cudaMemcpyAsync(dst, slabs[q], sizeof(double) * batch * pw, cudaMemcpyDefault, p.stream), "stage copy");
    } else {
      ck(cudaMemcpy2DAsync(dst, pw * sizeof(double), slabs[q], stride * sizeof(double), pw * sizeof(double), batch,
                           cudaMemcpyDefault, p.stream),
         "stage copy");
    }
  }
  const int64_t n = static_cast<int64_t>(p.Q) * batch * pw;
  k_stage<<<grid_for(n, 256, p.sms), 256, 0, p.stream>>>(p.stage, p.arena, p.G, p.top, batch, pw);
  ck(cudaGetLastError(), "stage launch");
}

// ---- sharding one polynomial across devices --------------------------------
int64_t exchange_words(const Plan& p, int rank, int batch) {
  if (p.nranks < 2) throw std::invalid_argument("plan is not sharded");
  if (rank < 0 || rank >= p.nranks) throw std::invalid_argument("bad rank");
  return static_cast<int64_t>(batch) * p.xslots[rank].second * p.G.slot_words;
}

// pack this rank's addition-stage slots (PACK) or write rank src's block into
// the arena (!PACK); buf is device memory, the call is stream-ordered and
// synchronous
template <bool PACK>
void exchange(Plan& p, int batch, int rank, double* buf) {
  if (batch < 1 || batch > p.max_batch) throw std::invalid_argument("batch outside [1, max_batch]");
  const int64_t n = exchange_words(p, rank, batch);
  ck(cudaSetDevice(p.device), "cudaSetDevice");
  if (n > 0) {
    if (!buf) throw std::invalid_argument("null exchange buffer");
    k_exchange<PACK><<<grid_for(n, 256, p.sms), 256, 0, p.stream>>>(p.arena, buf, p.G, p.xslots[rank].first,
                                                                    p.xslots[rank].second, batch);
    ck(cudaGetLastError(), "exchange launch");
  }
  ck(cudaStreamSynchronize(p.stream), "exchange");
}

// copy every peer's addition-stage slots from its arena (peer_arena) into
// ours; synchronous on the plan's stream. The peer table is uploaded once
// (and again only after a peer changes), so a gather is one kernel launch.
void gather_peers(Plan& p, int batch) {
  if (p.nranks < 2) throw std::invalid_argument("plan is not sharded");
  if (batch < 1 || batch > p.max_batch) throw std::invalid_argument("batch outside [1, max_batch]");
  ck(cudaSetDevice(p.device), "cudaSetDevice");
  if (p.peers_dirty) {
    std::vector<PeerList> peers;
    std::vector<int64_t> first(1, 0);
    for (int r = 0; r < p.nranks; ++r) {
      if (r == p.rank || p.xslots[r].second == 0) continue;
      if (r >= static_cast<int>(p.peer_arena.size()) || !p.peer_arena[r])
        throw std::invalid_argument("peer arena of rank " + std::to_string(r) + " not set");
      peers.push_back({p.peer_arena[r], p.xslots[r].first, p.xslots[r].second});
      first.push_back(first.back() + static_cast<int64_t>(p.xslots[r].second) * p.G.slot_words);
    }
    ck(cudaStreamSynchronize(p.stream), "peer table");
    cudaFree(p.peer_list);
    cudaFree(p.peer_first);
    p.peer_list = dev_upload(peers, p.stream);
    p.peer_first = dev_upload(first, p.stream);
    p.npeer_list = static_cast<int>(peers.size());
    p.peer_words1 = first.back();
    p.peers_dirty = false;
  }
  if (p.npeer_list == 0) return;
  k_gather_peers<<<grid_for(p.peer_words1 * batch, 256, p.sms), 256, 0, p.stream>>>(p.arena, p.G, p.peer_list,
                                                                                   p.npeer_list, p.peer_first, batch);
  ck(cudaGetLastError(), "peer gather launch");
  ck(cudaStreamSynchronize(p.stream), "peer gather");
}

// the addition stage of a sharded plan once every rank's slots are in place
int finish(Plan& p, int batch, int detail, pse_report* rep) {
  if (p.nranks < 2) throw std::invalid_argument("plan is not sharded");
  if (batch < 1 || batch > p.max_batch) throw std::invalid_argument("batch outside [1, max_batch]");
  ck(cudaSetDevice(p.device), "cudaSetDevice");
  p.ensure_events(2);
  (void)detail;
  ck(cudaEventRecord(p.ev[0], p.stream), "event");
  const int launches = p.launch_tail(batch);
  ck(cudaEventRecord(p.ev[1], p.stream), "event");
  ck(cudaGetLastError(), "launch");
  ck(cudaEventSynchronize(p.ev[1]), "finish");
  if (rep) {
    std::memset(rep, 0, sizeof *rep);
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, p.ev[0], p.ev[1]), "elapsed");
    p.read_stamps(rep, true);
    rep->device_ms = ms;
    rep->exchange_ms = p.exchange_ms;
    rep->kernel_launches = launches;
    rep->batch = batch;
  }
  return PSE_OK;
}

// One evaluation of the resident arena: the whole phase sequence is captured
// once per batch size into a CUDA graph and replayed. device_ms = CUDA events
// on the plan's stream around the replay; the phase times come from the
// kernels' own stamps of the same launches (read back when rep is given).
// detail is accepted for compatibility: every run is stamped.
int execute(Plan& p, int batch, int detail, pse_report* rep) {
  (void)detail;
  if (batch < 1 || batch > p.max_batch) throw std::invalid_argument("batch outside [1, max_batch]");
  ck(cudaSetDevice(p.device), "cudaSetDevice");
  p.ensure_events(2);
  p.prepare_band(batch);
  auto it = p.graphs.find(batch);
  if (it == p.graphs.end()) {
    cudaGraph_t graph;
    ck(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal), "capture");
    p.launch_all(batch);
    ck(cudaStreamEndCapture(p.stream, &graph), "capture end");
    cudaGraphExec_t exec;
    ck(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
    cudaGraphDestroy(graph);
    it = p.graphs.emplace(batch, exec).first;
  }
  ck(cudaEventRecord(p.ev[0], p.stream), "event");
  ck(cudaGraphLaunch(it->second, p.stream), "graph launch");
  ck(cudaEventRecord(p.ev[1], p.stream), "event");
  ck(cudaEventSynchronize(p.ev[1]), "execute");
  if (rep) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, p.ev[0], p.ev[1]), "elapsed");
    p.read_stamps(rep, p.nranks == 1);
    rep->device_ms = ms;
    fill_report(p, batch, rep);
    rep->kernel_launches = p.kernel_count(batch);
  }
  return PSE_OK;
}

void download(Plan& p, int batch, double* const* vg_out, double* const* dyn_out) {
  if (batch < 1 || batch > p.max_batch) throw std::invalid_argument("batch outside [1, max_batch]");
  ck(cudaSetDevice(p.device), "cudaSetDevice");
  const int64_t vw = static_cast<int64_t>(batch) * p.nrows * (p.d + 1);
  if (vg_out)
    for (int q = 0; q < p.Q; ++q)
      ck(cudaMemcpyAsync(vg_out[q], p.vg + static_cast<int64_t>(q) * vw, vw * sizeof(double),
                         cudaMemcpyDeviceToHost, p.stream),
         "D2H");
  if (dyn_out) {
    const int64_t dw = static_cast<int64_t>(batch) * p.TS * (p.d + 1);
    if (!p.dyn) p.dyn = dev_alloc<double>(static_cast<size_t>(p.Q) * p.max_batch * p.TS * (p.d + 1));
    const int64_t n = static_cast<int64_t>(p.Q) * dw;
    k_export<<<grid_for(n, 256, p.sms), 256, 0, p.stream>>>(p.arena, p.dyn, p.G, p.TS, batch);
    ck(cudaGetLastError(), "export launch");
    for (int q = 0; q < p.Q; ++q)
      ck(cudaMemcpyAsync(dyn_out[q], p.dyn + static_cast<int64_t>(q) * dw, dw * sizeof(double),
                         cudaMemcpyDeviceToHost, p.stream),
         "D2H");
  }
  ck(cudaStreamSynchronize(p.stream), "download");
}

// fold_exponents (jobgraph.cpp:168-197) as prologue conv jobs: for each
// monomial with exponents, folded = a_k; for each position j with e_j > 1:
// power = z (then power = conv(power, z), e_j - 2 times); folded =
// conv(folded, power). The final folded series is copied into a_k's slot,
// exactly where the reference stages it.
std::vector<std::vector<ConvRow>> fold_prologue(const HostGraph& hg, int64_t first_scratch, int64_t* nslots) {
  std::vector<std::vector<ConvRow>> layers;
  int64_t next = first_scratch;
  auto put = [&](size_t layer, ConvRow r) {
    if (layers.size() <= layer) layers.resize(layer + 1);
    layers[layer].push_back(r);
  };
  for (int k = 0; k < hg.N; ++k) {
    if (!hg.has_exponents(k)) continue;
    int64_t folded = 1 + k;
    size_t ready = 0;  // first layer at which `folded` is readable
    bool any = false;
    for (int64_t p = hg.mono_start[k]; p < hg.mono_start[k + 1]; ++p) {
      const int e = hg.exponents[p];
      if (e <= 1) continue;
      const int64_t z = hg.N + hg.indices[p];
      int64_t power = z;
      size_t pready = 0;
      for (int q = 2; q <= e - 1; ++q) {
        const int64_t out = next++;
        put(pready, {power, z, out, 0});
        power = out;
        ++pready;
      }
      const int64_t out = next++;
      const size_t L = std::max(ready, pready);
      put(L, {folded, power, out, 0});
      folded = out;
      ready = L + 1;
      any = true;
    }
    if (any) put(ready, {folded, 0, 1 + k, 1});
  }
  *nslots = next - first_scratch;
  return layers;
}

}  // namespace
}  // namespace pse

struct pse_plan {
  std::unique_ptr<pse::Plan> p;
};

extern "C" {

int pse_plan_create(const pse_graph_desc* desc, int32_t device, int32_t max_batch, pse_plan** out) {
  return pse::guarded([&] {
    if (!desc || !out) throw std::invalid_argument("null argument");
    auto* h = new pse_plan;
    h->p.reset(pse::build_plan(*desc, device, max_batch, {}, 0));
    *out = h;
    return PSE_OK;
  });
}

void pse_plan_destroy(pse_plan* p) { delete p; }

int pse_plan_create_sharded(const pse_graph_desc* desc, int32_t device, int32_t max_batch, int32_t rank,
                            int32_t nranks, pse_plan** out) {
  return pse::guarded([&] {
    if (!desc || !out) throw std::invalid_argument("null argument");
    auto* h = new pse_plan;
    h->p.reset(pse::build_plan(*desc, device, max_batch, {}, 0, rank, nranks));
    *out = h;
    return PSE_OK;
  });
}

int pse_plan_exchange_words(const pse_plan* p, int32_t rank, int32_t batch, int64_t* words) {
  return pse::guarded([&] {
    if (!p || !words) throw std::invalid_argument("null argument");
    *words = pse::exchange_words(*p->p, rank, batch);
    return PSE_OK;
  });
}

int pse_plan_pack(pse_plan* p, int32_t batch, double* dst) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    pse::exchange<true>(*p->p, batch, p->p->rank, dst);
    return PSE_OK;
  });
}

int pse_plan_unpack(pse_plan* p, int32_t batch, int32_t src_rank, const double* src) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    if (src_rank == p->p->rank) return PSE_OK;  // own slots are already in place
    pse::exchange<false>(*p->p, batch, src_rank, const_cast<double*>(src));
    return PSE_OK;
  });
}

int pse_plan_arena_ipc_handle(const pse_plan* p, void* handle) {
  return pse::guarded([&] {
    if (!p || !handle) throw std::invalid_argument("null argument");
    pse::ck(cudaSetDevice(p->p->device), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    pse::ck(cudaIpcGetMemHandle(&h, p->p->arena), "cudaIpcGetMemHandle");
    static_assert(sizeof h == PSE_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof h);
    return PSE_OK;
  });
}

static void set_peer(pse::Plan& P, int rank, const double* ptr, bool ipc) {
  if (P.nranks < 2) throw std::invalid_argument("plan is not sharded");
  if (rank < 0 || rank >= P.nranks || rank == P.rank) throw std::invalid_argument("bad peer rank");
  P.peer_arena.resize(P.nranks, nullptr);
  P.peer_ipc.resize(P.nranks, false);
  if (P.peer_ipc[rank] && P.peer_arena[rank]) cudaIpcCloseMemHandle(const_cast<double*>(P.peer_arena[rank]));
  P.peer_arena[rank] = ptr;
  P.peer_ipc[rank] = ipc;
  P.peers_dirty = true;
}

int pse_plan_open_peer(pse_plan* p, int32_t rank, const void* handle) {
  return pse::guarded([&] {
    if (!p || !handle) throw std::invalid_argument("null argument");
    pse::ck(cudaSetDevice(p->p->device), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void* ptr = nullptr;
    pse::ck(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    set_peer(*p->p, rank, static_cast<const double*>(ptr), true);
    return PSE_OK;
  });
}

int pse_plan_set_peer_arena(pse_plan* p, int32_t rank, const pse_plan* peer) {
  return pse::guarded([&] {
    if (!p || !peer) throw std::invalid_argument("null argument");
    if (peer->p->TSdev != p->p->TSdev || peer->p->G.point_words != p->p->G.point_words)
      throw std::invalid_argument("peer plan has a different arena geometry");
    if (peer->p->device != p->p->device) {  // direct peer access between devices of this process
      int ok = 0;
      pse::ck(cudaDeviceCanAccessPeer(&ok, p->p->device, peer->p->device), "cudaDeviceCanAccessPeer");
      if (!ok) throw std::invalid_argument("no peer access between the devices");
      pse::ck(cudaSetDevice(p->p->device), "cudaSetDevice");
      const cudaError_t e = cudaDeviceEnablePeerAccess(peer->p->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) pse::ck(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
    }
    set_peer(*p->p, rank, peer->p->arena, false);
    return PSE_OK;
  });
}

int pse_plan_gather_peers(pse_plan* p, int32_t batch) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    pse::gather_peers(*p->p, batch);
    return PSE_OK;
  });
}

int pse_plan_finish(pse_plan* p, int32_t batch, int32_t detail, pse_report* rep) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    return pse::finish(*p->p, batch, detail, rep);
  });
}

int pse_plan_upload(pse_plan* p, int32_t batch, const double* const* static_slabs, int64_t point_stride) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    pse::upload(*p->p, batch, static_slabs, point_stride);
    pse::ck(cudaStreamSynchronize(p->p->stream), "upload");
    return PSE_OK;
  });
}

int pse_plan_execute(pse_plan* p, int32_t batch, int32_t detail, pse_report* rep) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    if (rep) std::memset(rep, 0, sizeof *rep);
    return pse::execute(*p->p, batch, detail, rep);
  });
}

int pse_plan_download(pse_plan* p, int32_t batch, double* const* value_grad_out, double* const* dyn_slabs_out) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    pse::download(*p->p, batch, value_grad_out, dyn_slabs_out);
    return PSE_OK;
  });
}

int pse_plan_run(pse_plan* p, int32_t batch, const double* const* static_slabs, int64_t point_stride,
                 double* const* dyn_slabs_out, double* const* value_grad_out, pse_report* rep) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    pse::Plan& P = *p->p;
    pse::ck(cudaSetDevice(P.device), "cudaSetDevice");
    P.ensure_events(6);  // ev[0..1]: execute; ev[2..5]: this call
    pse::ck(cudaEventRecord(P.ev[2], P.stream), "event");
    pse::upload(P, batch, static_slabs, point_stride);
    pse::ck(cudaEventRecord(P.ev[3], P.stream), "event");
    pse_report r{};
    pse::execute(P, batch, 0, &r);
    pse::ck(cudaEventRecord(P.ev[4], P.stream), "event");
    pse::download(P, batch, value_grad_out, dyn_slabs_out);
    pse::ck(cudaEventRecord(P.ev[5], P.stream), "event");
    pse::ck(cudaEventSynchronize(P.ev[5]), "run");
    float h2d = 0, d2h = 0, all = 0;
    pse::ck(cudaEventElapsedTime(&h2d, P.ev[2], P.ev[3]), "elapsed");
    pse::ck(cudaEventElapsedTime(&d2h, P.ev[4], P.ev[5]), "elapsed");
    pse::ck(cudaEventElapsedTime(&all, P.ev[2], P.ev[5]), "elapsed");
    r.h2d_ms = h2d;
    r.d2h_ms = d2h;
    r.e2e_ms = all;
    r.kernel_launches += 1 + (dyn_slabs_out ? 1 : 0);
    if (rep) *rep = r;
    return PSE_OK;
  });
}

int pse_plan_layer_ms(const pse_plan* p, double* conv_layer_ms, int32_t n_conv, double* add_layer_ms, int32_t n_add) {
  return pse::guarded([&] {
    if (!p) throw std::invalid_argument("null plan");
    const pse::Plan& P = *p->p;
    if (n_conv != P.n_conv_layers || n_add != P.n_add_layers)
      throw std::invalid_argument("layer counts do not match the plan's graph");
    if ((n_conv && !conv_layer_ms) || (n_add && !add_layer_ms)) throw std::invalid_argument("null argument");
    for (int l = 0; l < n_conv; ++l) conv_layer_ms[l] = l < static_cast<int>(P.conv_layer_ms.size()) ? P.conv_layer_ms[l] : 0.0;
    for (int l = 0; l < n_add; ++l) add_layer_ms[l] = l < static_cast<int>(P.add_layer_ms.size()) ? P.add_layer_ms[l] : 0.0;
    return PSE_OK;
  });
}

int pse_plan_stream(const pse_plan* p, void** stream) {
  if (!p || !stream) return PSE_EINVAL;
  *stream = p->p->stream;
  return PSE_OK;
}

int pse_plan_conv_path(const pse_plan* p, int32_t batch, int32_t* path) {
  if (!p || !path || batch < 1 || batch > p->p->max_batch) return PSE_EINVAL;
  const pse::Plan& P = *p->p;
  *path = !P.banded(batch)          ? PSE_CONV_LAYERED
          : P.cta_mode()            ? (P.cta.layered ? PSE_CONV_CTA_LAYERS : PSE_CONV_CTA)
          : !P.flow()               ? PSE_CONV_WAVES
          : P.band_first(batch) > 0 ? PSE_CONV_HYBRID
                                    : PSE_CONV_DATAFLOW;
  return PSE_OK;
}

int pse_band_schedule_stats(const pse_graph_desc* desc, int32_t W, int32_t flow, int64_t procs, double slack,
                            int64_t* out) {
  return pse::guarded([&] {
    if (!desc || !out) throw std::invalid_argument("null argument");
    if (W != 16 && W != 32) throw std::invalid_argument("band width must be 16 or 32");
    if (procs < 1) throw std::invalid_argument("procs must be at least 1");
    const std::string why = pse::validate_desc(*desc);
    if (!why.empty()) throw std::invalid_argument("invalid job graph: " + why);
    int64_t next = desc->total_slots;
    const auto layers = pse::versioned_layers(*desc, {}, &next);
    std::vector<pse::ConvRow> rows;
    for (auto& l : layers) rows.insert(rows.end(), l.begin(), l.end());
    const pse::BandSched s = pse::band_schedule(rows, desc->d, W, pse::kSlots * procs, flow != 0, procs * (32 / W),
                                                slack, 1.0);
    int64_t descs = 0, tasks = 0, slots = 0;
    for (auto& w : s.waves) {
      descs += static_cast<int64_t>(w.size()) / pse::kSlots;
      for (size_t i = 0; i < w.size(); ++i) {
        if (w[i].w == -4) continue;
        ++slots;
        const int lanes = w[i].w == -2 ? W / 2 : W;
        if (static_cast<int>(i % pse::kSlots) % (lanes / 8) == 0) ++tasks;  // first slot of a task
      }
    }
    out[0] = static_cast<int64_t>(rows.size());
    out[1] = tasks;
    out[2] = descs;
    out[3] = static_cast<int64_t>(s.waves.size());
    out[4] = static_cast<int64_t>(s.deps.size());
    out[5] = slots;
    out[6] = static_cast<int64_t>(s.makespan);
    return PSE_OK;
  });
}

int pse_plan_info(const pse_plan* p, int64_t* out) {
  if (!p || !out) return PSE_EINVAL;
  const pse::Plan& P = *p->p;
  int64_t v[8] = {P.n, P.N, P.d, P.m, P.mode, P.TS, P.top, P.max_batch};
  std::memcpy(out, v, sizeof v);
  return PSE_OK;
}

int pse_evaluate(int32_t n, int32_t d, int32_t m, int32_t mode, int32_t N, const int32_t* nvars,
                 const int32_t* indices, const int32_t* exponents, int32_t batch, const double* stat,
                 double* vg_out, int32_t device, pse_report* rep) {
  return pse::guarded([&] {
    if (!nvars || !indices || !stat || !vg_out) throw std::invalid_argument("null argument");
    if (!pse::valid_precision(m)) throw std::invalid_argument("unsupported precision level");
    if (batch < 1) throw std::invalid_argument("batch must be at least 1");
    pse::HostGraph hg = pse::build_graph(n, d, N, nvars, indices, exponents);
    const pse_graph_desc desc = pse::describe(hg, m, mode);
    int64_t extra = 0;
    auto pro = pse::fold_prologue(hg, hg.total_slots, &extra);
    std::unique_ptr<pse::Plan> P(pse::build_plan(desc, device, batch, pro, extra));
    const int Q = P->Q;
    const int64_t pw = P->top * (d + 1);
    std::vector<const double*> slabs(Q);
    for (int q = 0; q < Q; ++q) slabs[q] = stat + static_cast<int64_t>(q) * batch * pw;
    const int64_t vw = static_cast<int64_t>(batch) * (n + 1) * (d + 1);
    std::vector<double*> outs(Q);
    for (int q = 0; q < Q; ++q) outs[q] = vg_out + q * vw;
    pse::upload(*P, batch, slabs.data(), pw);
    pse_report r{};
    pse::execute(*P, batch, 1, &r);
    pse::download(*P, batch, outs.data(), nullptr);
    if (rep) *rep = r;
    return PSE_OK;
  });
}

int pse_md_apply(int32_t op, int32_t m, int32_t impl, int64_t count, const double* x, const double* y, double* out,
                 int32_t device) {
  return pse::guarded([&] {
    if (!pse::valid_precision(m)) throw std::invalid_argument("unsupported precision level");
    if (op < 0 || op > 2 || count < 0) throw std::invalid_argument("bad md op");
    if (count == 0) return PSE_OK;
    pse::ck(cudaSetDevice(device), "cudaSetDevice");
    const size_t bytes = static_cast<size_t>(count) * m * sizeof(double);
    double *dx, *dy, *dz;
    pse::ck(cudaMalloc(&dx, bytes), "cudaMalloc");
    pse::ck(cudaMalloc(&dy, bytes), "cudaMalloc");
    pse::ck(cudaMalloc(&dz, bytes), "cudaMalloc");
    pse::ck(cudaMemcpy(dx, x, bytes, cudaMemcpyHostToDevice), "H2D");
    pse::ck(cudaMemcpy(dy, y, bytes, cudaMemcpyHostToDevice), "H2D");
    pse::MdArgs a{op, impl, count, dx, dy, dz};
    const pse::Launchers* L = pse::launchers_for(m, false);
    L->prepare();
    L->md(a, nullptr);
    pse::ck(cudaGetLastError(), "md launch");
    pse::ck(cudaMemcpy(out, dz, bytes, cudaMemcpyDeviceToHost), "D2H");
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dz);
    return PSE_OK;
  });
}

int pse_series_conv(int32_t d, int32_t m, int32_t mode, int64_t count, const double* x, const double* y, double* z,
                    int32_t device) {
  return pse::guarded([&] {
    if (!pse::valid_precision(m) || d < 0 || count < 0) throw std::invalid_argument("bad series arguments");
    if (count == 0) return PSE_OK;
    pse::ck(cudaSetDevice(device), "cudaSetDevice");
    const int Q = (mode == PSE_MODE_COMPLEX ? 2 : 1) * m;
    pse::Geom G;
    G.d = d;
    G.S = d + 1;
    G.Q = Q;
    G.slot_words = static_cast<int64_t>(Q) * G.S;
    G.point_words = 3 * G.slot_words;  // slots x, y, z per pair
    const size_t words = static_cast<size_t>(count) * G.point_words;
    double* arena;
    pse::ck(cudaMalloc(&arena, words * sizeof(double)), "cudaMalloc");
    const int64_t sw = G.slot_words;
    pse::ck(cudaMemcpy2D(arena, 3 * sw * sizeof(double), x, sw * sizeof(double), sw * sizeof(double), count,
                         cudaMemcpyHostToDevice),
            "H2D");
    pse::ck(cudaMemcpy2D(arena + sw, 3 * sw * sizeof(double), y, sw * sizeof(double), sw * sizeof(double), count,
                         cudaMemcpyHostToDevice),
            "H2D");
    int4* job;
    pse::ck(cudaMalloc(&job, sizeof(int4)), "cudaMalloc");
    const int4 hj = make_int4(0, 1, 2, 0);
    pse::ck(cudaMemcpy(job, &hj, sizeof hj, cudaMemcpyHostToDevice), "H2D");
    pse::ConvArgs a{arena, G, job, 1, (d + 2) / 2, static_cast<int>(count)};
    const pse::Launchers* L = pse::launchers_for(m, mode == PSE_MODE_COMPLEX);
    L->prepare();
    L->conv(a, nullptr);
    pse::ck(cudaGetLastError(), "conv launch");
    pse::ck(cudaMemcpy2D(z, sw * sizeof(double), arena + 2 * sw, 3 * sw * sizeof(double), sw * sizeof(double), count,
                         cudaMemcpyDeviceToHost),
            "D2H");
    cudaFree(job);
    cudaFree(arena);
    return PSE_OK;
  });
}

extern "C++" {
namespace pse {
// one-shot device run of a series primitive over `count` independent items of
// `nslots` series each (host layout [count][nslots][Q][d+1]); `launch` gets
// the arena and geometry, slot 0 comes back as the result
template <class F>
int series_oneshot(int32_t d, int32_t m, int32_t mode, int64_t count, int nslots, const double* const* in,
                   double* z, int32_t device, F&& launch) {
  if (!valid_precision(m) || d < 0 || count < 0 || count > (int64_t(1) << 31) / (d + 1))
    throw std::invalid_argument("bad series arguments");
  if (count == 0) return PSE_OK;
  ck(cudaSetDevice(device), "cudaSetDevice");
  Geom G;
  G.d = d;
  G.S = d + 1;
  G.Q = (mode == PSE_MODE_COMPLEX ? 2 : 1) * m;
  G.slot_words = static_cast<int64_t>(G.Q) * G.S;
  G.point_words = nslots * G.slot_words;
  const int64_t sw = G.slot_words;
  double* arena;
  ck(cudaMalloc(&arena, static_cast<size_t>(count) * G.point_words * sizeof(double)), "cudaMalloc");
  for (int sl = 0; sl < nslots; ++sl)
    ck(cudaMemcpy2D(arena + sl * sw, nslots * sw * sizeof(double), in[sl], sw * sizeof(double), sw * sizeof(double),
                    count, cudaMemcpyHostToDevice),
       "H2D");
  const Launchers* L = launchers_for(m, mode == PSE_MODE_COMPLEX);
  L->prepare();
  launch(L, arena, G);
  ck(cudaGetLastError(), "series launch");
  ck(cudaMemcpy2D(z, sw * sizeof(double), arena, nslots * sw * sizeof(double), sw * sizeof(double), count,
                  cudaMemcpyDeviceToHost),
     "D2H");
  cudaFree(arena);
  return PSE_OK;
}
}  // namespace pse
}  // extern "C++"

int pse_series_add(int32_t d, int32_t m, int32_t mode, int64_t count, const double* x, const double* y, double* z,
                   int32_t device) {
  return pse::guarded([&] {
    const double* in[2] = {x, y};
    return pse::series_oneshot(d, m, mode, count, 2, in, z, device, [&](const pse::Launchers* L, double* arena,
                                                                        const pse::Geom& G) {
      int2* job;
      pse::ck(cudaMalloc(&job, sizeof(int2)), "cudaMalloc");
      const int2 hj = make_int2(1, 0);  // slot 0 := md_add(slot 0, slot 1)
      pse::ck(cudaMemcpy(job, &hj, sizeof hj, cudaMemcpyHostToDevice), "H2D");
      pse::AddArgs a{arena, G, job, 1, static_cast<int>(count), nullptr, nullptr};
      L->add(a, nullptr);
      pse::ck(cudaDeviceSynchronize(), "series add");
      cudaFree(job);
    });
  });
}

int pse_series_scale_int(int32_t d, int32_t m, int32_t mode, int64_t count, const double* x, int64_t factor,
                         double* z, int32_t device) {
  return pse::guarded([&] {
    if (factor > INT32_MAX || factor < INT32_MIN) throw std::invalid_argument("factor out of range");
    const double* in[1] = {x};
    return pse::series_oneshot(d, m, mode, count, 1, in, z, device, [&](const pse::Launchers* L, double* arena,
                                                                        const pse::Geom& G) {
      int2* item;
      pse::ck(cudaMalloc(&item, sizeof(int2)), "cudaMalloc");
      const int2 hi = make_int2(0, static_cast<int>(factor));
      pse::ck(cudaMemcpy(item, &hi, sizeof hi, cudaMemcpyHostToDevice), "H2D");
      pse::ScaleArgs a{arena, G, item, 1, static_cast<int>(count), nullptr, nullptr};
      L->scale(a, nullptr);
      pse::ck(cudaDeviceSynchronize(), "series scale");
      cudaFree(item);
    });
  });
}

void* pse_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
    pse::set_error("cudaHostAlloc failed");
    return nullptr;
  }
  return p;
}

void pse_host_free(void* p) { cudaFreeHost(p); }

int pse_device_info(int32_t device, int64_t* out) {
  return pse::guarded([&] {
    int count = 0;
    pse::ck(cudaGetDeviceCount(&count), "device count");
    cudaDeviceProp prop;
    pse::ck(cudaGetDeviceProperties(&prop, device), "props");
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    out[0] = prop.multiProcessorCount;
    out[1] = clk;
    out[2] = prop.major * 10 + prop.minor;
    out[3] = count;
    return PSE_OK;
  });
}

}  // extern "C"
