// Native JSONL emitters for the trace and event-log formats (host code; no CUDA calls).
//
// Byte-identical to the reference's writers (json.dumps with separators (",", ":"), keys in
// the documented order, id lists ascending):
//   moe_format_trace      <- traces.write_trace        traces.py:267-312
//   moe_format_event_log  <- simulate.write_event_log  simulate.py:187-226 (+ steps(), :88-111)
// Lines are independent, so long traces are formatted in token chunks on all host threads and
// concatenated in order.
#include "common.cuh"

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

inline void put_int(std::string& s, long long v) {
  char buf[24];
  int n = 0;
  const bool neg = v < 0;
  unsigned long long u = neg ? 0ull - static_cast<unsigned long long>(v) : static_cast<unsigned long long>(v);
  do {
    buf[n++] = static_cast<char>('0' + u % 10);
    u /= 10;
  } while (u);
  if (neg) buf[n++] = '-';
  while (n) s.push_back(buf[--n]);
}

template <class I>
inline void put_list(std::string& s, const I* v, int n) {
  s.push_back('[');
  for (int i = 0; i < n; ++i) {
    if (i) s.push_back(',');
    put_int(s, v[i]);
  }
  s.push_back(']');
}

// Format tokens [t0, t1) with `fmt(t, out)` on up to hardware_concurrency threads; returns
// the chunks' concatenation.
template <class F>
std::string parallel_lines(long long T, long long lines_per_token, F fmt) {
  const long long total = T * lines_per_token;
  unsigned nth = std::max(1u, std::thread::hardware_concurrency());
  if (total < 65536) nth = 1;
  nth = static_cast<unsigned>(std::min<long long>(nth, std::max<long long>(1, T)));
  std::vector<std::string> parts(nth);
  auto run = [&](unsigned i) {
    const long long a = T * i / nth, b = T * (i + 1) / nth;
    std::string& s = parts[i];
    s.reserve(static_cast<size_t>((b - a) * lines_per_token * 48));
    for (long long t = a; t < b; ++t) fmt(t, s);
  };
  if (nth == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nth; ++i) th.emplace_back(run, i);
    for (auto& x : th) x.join();
  }
  size_t n = 0;
  for (auto& p : parts) n += p.size();
  std::string out;
  out.reserve(n);
  for (auto& p : parts) out += p;
  return out;
}

}  // namespace

struct moe_text {
  std::string s;
};

namespace {
moe_status emit(std::string&& body, const std::string& head, moe_text** doc) {
  auto* d = new moe_text();
  d->s.reserve(head.size() + body.size());
  d->s += head;
  d->s += body;
  *doc = d;
  return MOE_OK;
}
}  // namespace

extern "C" {

const char* moe_text_data(const moe_text* doc) { return doc ? doc->s.data() : nullptr; }
int64_t moe_text_size(const moe_text* doc) { return doc ? static_cast<int64_t>(doc->s.size()) : 0; }
void moe_text_free(moe_text* doc) { delete doc; }

moe_status moe_format_trace(int32_t kind, int32_t num_layers, int32_t num_experts, int32_t top_k,
                            int64_t T, const int64_t* grid_a, const int64_t* grid_g,
                            moe_text** doc) {
  MOE_REQUIRE(doc, "null doc");
  MOE_REQUIRE(kind == 0 || kind == 1, "kind must be 0 (activation) or 1 (speculation)");
  MOE_REQUIRE(T >= 0 && num_layers >= 1 && top_k >= 1, "bad trace shape");
  MOE_REQUIRE(T == 0 || grid_a, "null activation grid");
  MOE_REQUIRE(kind == 0 || T == 0 || num_layers < 2 || grid_g, "null guess grid");
  const int L = num_layers, K = top_k;
  std::string head = kind == 0 ? "{\"kind\":\"activation\",\"num_layers\":" : "{\"kind\":\"speculation\",\"num_layers\":";
  put_int(head, L);
  head += ",\"num_experts\":";
  put_int(head, num_experts);
  head += ",\"top_k\":";
  put_int(head, K);
  head += "}\n";
  std::string body;
  if (kind == 0) {
    body = parallel_lines(T, L, [&](long long t, std::string& s) {
      for (int l = 0; l < L; ++l) {
        s += "{\"t\":";
        put_int(s, t);
        s += ",\"l\":";
        put_int(s, l);
        s += ",\"a\":";
        put_list(s, grid_a + (t * L + l) * K, K);
        s += "}\n";
      }
    });
  } else {
    const int J = L - 1;  // (T, L-1, K) grids, records for layers 1..L-1
    body = parallel_lines(T, std::max(J, 0), [&](long long t, std::string& s) {
      for (int j = 0; j < J; ++j) {
        s += "{\"t\":";
        put_int(s, t);
        s += ",\"l\":";
        put_int(s, j + 1);
        s += ",\"g\":";
        put_list(s, grid_g + (t * J + j) * K, K);
        s += ",\"a\":";
        put_list(s, grid_a + (t * J + j) * K, K);
        s += "}\n";
      }
    });
  }
  return emit(std::move(body), head, doc);
}

// Event log: layers[n_layers] are the replayed layer ids (log.layers); activated
// (n_layers, T, K) int64, resident_before / evicted (n_layers, T, E) uint8 -- the columnar
// CacheEventLog.  Steps in (token, layer) order; cached / hit / miss / evict ascending, hit
// and miss as sets (activations & resident_before, activations - resident_before).
moe_status moe_format_event_log(const char* policy, int32_t cache_size, int32_t num_layers,
                                int32_t num_experts, int32_t top_k, int64_t warmup_tokens,
                                int32_t n_layers, const int32_t* layers, int64_t T,
                                const int64_t* activated, const uint8_t* resident_before,
                                const uint8_t* evicted, moe_text** doc) {
  MOE_REQUIRE(doc && policy, "null argument");
  MOE_REQUIRE(T >= 0 && n_layers >= 0 && num_experts >= 1 && top_k >= 1, "bad event-log shape");
  MOE_REQUIRE(T == 0 || n_layers == 0 || (layers && activated && resident_before && evicted),
              "null event-log arrays");
  const int E = num_experts, K = top_k, NL = n_layers;
  std::string head = "{\"kind\":\"events\",\"policy\":\"";
  head += policy;
  head += "\",\"cache_size\":";
  put_int(head, cache_size);
  head += ",\"num_layers\":";
  put_int(head, num_layers);
  head += ",\"num_experts\":";
  put_int(head, E);
  head += ",\"top_k\":";
  put_int(head, K);
  head += ",\"warmup_tokens\":";
  put_int(head, warmup_tokens);
  head += "}\n";
  std::string body = parallel_lines(T, NL, [&](long long t, std::string& s) {
    std::vector<long long> ids;
    ids.reserve(E);
    std::vector<char> in_act(E);
    for (int i = 0; i < NL; ++i) {
      const int64_t* a = activated + (static_cast<long long>(i) * T + t) * K;
      const uint8_t* rb = resident_before + (static_cast<long long>(i) * T + t) * E;
      const uint8_t* ev = evicted + (static_cast<long long>(i) * T + t) * E;
      std::fill(in_act.begin(), in_act.end(), 0);
      for (int j = 0; j < K; ++j)
        if (a[j] >= 0 && a[j] < E) in_act[a[j]] = 1;
      s += "{\"t\":";
      put_int(s, t);
      s += ",\"l\":";
      put_int(s, layers[i]);
      s += ",\"cached\":";
      ids.clear();
      for (int e = 0; e < E; ++e)
        if (rb[e]) ids.push_back(e);
      put_list(s, ids.data(), static_cast<int>(ids.size()));
      s += ",\"hit\":";
      ids.clear();
      for (int e = 0; e < E; ++e)
        if (in_act[e] && rb[e]) ids.push_back(e);
      put_list(s, ids.data(), static_cast<int>(ids.size()));
      s += ",\"miss\":";
      ids.clear();
      for (int e = 0; e < E; ++e)
        if (in_act[e] && !rb[e]) ids.push_back(e);
      put_list(s, ids.data(), static_cast<int>(ids.size()));
      s += ",\"evict\":";
      ids.clear();
      for (int e = 0; e < E; ++e)
        if (ev[e]) ids.push_back(e);
      put_list(s, ids.data(), static_cast<int>(ids.size()));
      s += "}\n";
    }
  });
  return emit(std::move(body), head, doc);
}

}  // extern "C"
