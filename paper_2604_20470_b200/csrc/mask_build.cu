// Mask builder entry points (stub; filled in by the next milestone).
#include "internal.hpp"
#include "plan.hpp"

using namespace rp;

struct rp_plan_s {
  rp_grid g;
  rp_config c;
  uint64_t seed;
  rp_build_options o;
};

extern "C" {
void rp_build_options_defaults(rp_build_options* o) {
  o->disable_split = 0;
  o->score_engine = 0;
  o->recheck_delta = 0.0;
}
rp_status rp_plan_create(const rp_grid* g, const rp_config* c, uint64_t seed,
                         const rp_build_options* opt, rp_plan* out) {
  return guarded([&] {
    check_grid(g);
    plan::validate(*c);
    auto* p = new rp_plan_s{*g, *c, seed, {}};
    if (opt) p->o = *opt; else rp_build_options_defaults(&p->o);
    *out = p;
  });
}
void rp_plan_destroy(rp_plan p) { delete p; }
rp_status rp_plan_build_mask(rp_plan, const rp_tensor*, const rp_tensor*, int, uint8_t*,
                             rp_build_stats*, rp_stream) {
  return guarded([&] { throw std::runtime_error("rp_plan_build_mask: not implemented yet"); });
}
rp_status rp_build_mask(const rp_grid* g, const rp_config* c, uint64_t seed,
                        const rp_build_options* opt, const rp_tensor* q, const rp_tensor* k,
                        int n, uint8_t* bits, rp_build_stats* st, rp_stream s) {
  rp_plan p = nullptr;
  rp_status r = rp_plan_create(g, c, seed, opt, &p);
  if (r != RP_OK) return r;
  r = rp_plan_build_mask(p, q, k, n, bits, st, s);
  rp_plan_destroy(p);
  return r;
}
}
