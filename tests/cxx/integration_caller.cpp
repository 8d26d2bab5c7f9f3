// A reference-style C++ caller linked against libhlm_b200.so through the C++ API in
// include/hlm/*.hpp — the shape of the reference's own call sites
// (proj/tools/hlm_main.cpp:191-236 cmd_train, proj/src/trainer.cpp:8-42,
// proj/tests/test_engine.cpp phase-API tests). INTEGRATION.md §1 quotes it.
//
//   integration_caller train  L h f V S B K heads steps   -> one "loss <hex> <value>" line per step
//   integration_caller trainx ...                          -> the same with bench.py's scheduling features
//   integration_caller phases L h f V S B K heads          -> loss of one step via the phase API
//   integration_caller errors                              -> exercises the exception mapping
//   integration_caller arena                               -> DeviceArena / ledger contract
//                                                             (reference proj/tests/test_arena.cpp:160-215)
//   integration_caller ledger L h f V S B K heads           -> footprint vs the live ledger after one step
//                                                             (reference proj/tests/test_planner.cpp:43-72)
//   integration_caller hlm1 in out L h f V S B K heads      -> load_checkpoint of a reference HLM1 file,
//                                                             save_checkpoint_hlm1 back (host only, no GPU)
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "hlm/checkpoint.hpp"
#include "hlm/engine.hpp"
#include "hlm/trainer.hpp"

namespace {

hlm::ModelConfig config_from(char** a) {
    hlm::ModelConfig m;
    m.layers = std::atoll(a[0]);
    m.hidden = std::atoll(a[1]);
    m.ffn = std::atoll(a[2]);
    m.vocab = std::atoll(a[3]);
    m.seq = std::atoll(a[4]);
    m.batch = std::atoll(a[5]);
    m.k_ckpt = std::atoll(a[6]);
    m.n_heads = std::atoi(a[7]);
    m.rope_theta = m.n_heads > 1 ? 1e6 : 0.0;
    return m;
}

void print_loss(double loss) {
    std::uint64_t bits;
    std::memcpy(&bits, &loss, sizeof bits);
    std::printf("loss %016" PRIx64 " %.9g\n", bits, loss);
}

int train(char** a, bool bench_features = false) {
    hlm::RunConfig cfg;
    cfg.model = config_from(a);
    cfg.model.validate();
    cfg.run.steps = std::atoll(a[8]);
    cfg.run.seed = 1234;
    cfg.run.eager_optim = true;
    cfg.run.threaded_accum = true;
    cfg.run.n_slab = 3;
    cfg.hyper.lr = 3e-3;
    auto store = hlm::build_store(cfg.model, cfg.run.seed, hlm::Dtype::BF16, hlm::InitMode::Reference);
    hlm::EngineOptions opts;   // `trainx`: bench.py's feature set (every host thread hand-off)
    hlm::i64 cache = 0;
    if (bench_features) {
        opts.overlap_optimizer_tail = true;
        opts.tail_blocks = 2;
        opts.piece_elems = 4096;
        opts.grad_buffers = 4;
        opts.sparse_embed_grad = true;
        opts.embed_gather_host = true;
        opts.head_piece_vocab = 128;
        cache = 2 * (2 * cfg.model.block_params() + 255) / 256 * 256;
    }
    hlm::DeviceArena arena(cfg.model, std::nullopt, -1, cache);
    const hlm::TrainOutput out =
        hlm::run_training(cfg, *store, arena, [](const hlm::StepTelemetry& t) { print_loss(t.loss); }, opts);
    std::printf("h2d %" PRId64 " d2h %" PRId64 " steps %" PRId64 "\n", out.steps.back().h2d_bytes,
                out.steps.back().d2h_bytes, store->adam_steps());
    return 0;
}

int phases(char** a) {
    const hlm::ModelConfig m = config_from(a);
    auto store = hlm::build_store(m, 1234, hlm::Dtype::BF16, hlm::InitMode::Reference);
    hlm::DeviceArena arena(m);
    hlm::EngineOptions opts;
    opts.skip_optimizer = true;
    hlm::Engine engine(*store, arena, hlm::HyperParams{}, opts);
    hlm::Rng data(1235);
    engine.begin_step(hlm::make_copy_task_batch(m, data));
    engine.forward_streaming();
    const double loss = engine.anchor_loss();
    engine.backward_blockwise();
    const hlm::StepResult r = engine.finish_step();
    print_loss(loss);
    print_loss(r.loss);
    std::printf("recompute_forwards %" PRId64 "\n", r.recompute_forwards);
    return 0;
}

// The reference's error contract (errors.hpp:13-50, hlm_main.cpp:418-430) across the
// shared-library boundary: the exception types thrown inside libhlm_b200.so are
// caught by their C++ type here.
int errors() {
    hlm::ModelConfig m;
    m.layers = 2; m.hidden = 64; m.ffn = 128; m.vocab = 64; m.seq = 32; m.batch = 2; m.k_ckpt = 1;
    int seen = 0;
    try {
        hlm::ModelConfig bad = m;
        bad.hidden = 0;
        bad.validate();
    } catch (const std::invalid_argument& e) {   // model_config.hpp:28-40
        std::printf("invalid_argument: %s\n", e.what());
        ++seen;
    }
    try {
        hlm::DeviceArena tiny(m, std::optional<hlm::i64>(4096));
    } catch (const hlm::ArenaOomError& e) {
        std::printf("ArenaOomError region=%s requested=%" PRId64 " capacity=%" PRId64 "\n",
                    e.region().c_str(), e.requested(), e.capacity());
        ++seen;
    }
    auto store = hlm::build_store(m, 7, hlm::Dtype::BF16);
    hlm::DeviceArena arena(m);
    hlm::Engine engine(*store, arena, hlm::HyperParams{});
    try {
        engine.forward_streaming();   // before begin_step
    } catch (const hlm::ProtocolError& e) {
        std::printf("ProtocolError: %s\n", e.what());
        ++seen;
    }
    try {
        hlm::Batch b;
        b.tokens.assign(static_cast<size_t>(m.batch * m.seq), 0);
        b.targets = b.tokens;
        b.tokens[5] = static_cast<std::int32_t>(m.vocab);   // out of range
        engine.train_step(b);
    } catch (const std::out_of_range& e) {
        std::printf("out_of_range: %s\n", e.what());
        ++seen;
    }
    std::printf("errors caught %d\n", seen);
    return seen == 4 ? 0 : 1;
}

int failures = 0;
void expect(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "ok" : "FAIL", what);
    if (!ok) ++failures;
}

template <typename Ex, typename F>
bool throws(F&& f) {
    try {
        f();
    } catch (const Ex&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int arena() {
    hlm::ModelConfig m;
    m.layers = 8; m.hidden = 64; m.ffn = 128; m.vocab = 64; m.seq = 32; m.batch = 2; m.k_ckpt = 2;
    const hlm::ArenaFootprint fp = hlm::arena_footprint(m);
    expect(!throws<std::exception>([&] { hlm::DeviceArena a(m, fp.total()); }), "an exact budget cap fits");
    try {
        hlm::DeviceArena a(m, fp.total() - 1);
        expect(false, "budget cap total-1 throws");
    } catch (const hlm::ArenaOomError& e) {
        expect(e.region() == "workspace", "budget cap total-1 names the last region to claim (workspace)");
    }
    try {
        hlm::DeviceArena a(m, 16);
        expect(false, "budget cap 16 throws");
    } catch (const hlm::ArenaOomError& e) {
        expect(e.region() == "stream_buf[0]", "budget cap 16 names stream_buf[0]");
    }
    hlm::DeviceArena arena(m);
    arena.begin_step();
    const hlm::i64 start = arena.ledger().current(hlm::Region::Stack);
    arena.push_acts();
    arena.push_acts();   // capacity: K = 2 slabs
    expect(arena.ledger().current(hlm::Region::Stack) == start + fp.stack, "two pushes fill the K-slab stack");
    try {
        arena.push_acts();
        expect(false, "third push throws");
    } catch (const hlm::ArenaOomError& e) {
        expect(e.region() == "activation_stack" && e.requested() > e.capacity(),
               "stack overflow is an OOM naming activation_stack, requested > capacity");
    }
    arena.pop_acts();
    arena.pop_acts();
    expect(arena.ledger().current(hlm::Region::Stack) == start, "pops return the stack to its start");
    expect(throws<hlm::ProtocolError>([&] { arena.pop_acts(); }), "pop of an empty stack is a ProtocolError");
    arena.anchor_checkpoint(0);
    arena.anchor_checkpoint(4);
    arena.anchor_checkpoint(8);
    expect(arena.ledger().current(hlm::Region::Anchors) == 3 * fp.anchor_slot, "three anchors claimed");
    expect(throws<hlm::ProtocolError>([&] { arena.load_checkpoint(6); }), "never-anchored load throws");
    expect(throws<hlm::ProtocolError>([&] { arena.anchor_checkpoint(3); }), "anchor off the K grid throws");
    arena.release_checkpoint(4);
    expect(throws<hlm::ProtocolError>([&] { arena.load_checkpoint(4); }), "released anchor cannot be loaded");
    arena.release_checkpoint(0);
    arena.release_checkpoint(8);
    expect(arena.ledger().current(hlm::Region::Anchors) == 0, "anchors released");
    expect(throws<hlm::ProtocolError>([&] {
               arena.claim_buffer(0, 1, 8);
               arena.claim_buffer(0, 2, 8);
           }),
           "stream_in into a busy buffer is a ProtocolError");
    std::printf("arena failures %d\n", failures);
    return failures ? 1 : 0;
}

int ledger(char** a) {
    const hlm::ModelConfig m = config_from(a);
    auto store = hlm::build_store(m, 1234, hlm::Dtype::BF16, hlm::InitMode::Reference);
    hlm::DeviceArena arena(m);
    hlm::EngineOptions opts;
    opts.eager_optim = true;
    opts.threaded_accum = true;
    opts.n_slab = 4;
    hlm::Engine engine(*store, arena, hlm::HyperParams{}, opts);
    hlm::Rng data(1235);
    const hlm::StepResult r = engine.train_step(hlm::make_copy_task_batch(m, data));
    const hlm::ArenaFootprint fp = hlm::arena_footprint(m);
    std::printf("footprint total %" PRId64 " core %" PRId64 " anchors %" PRId64 " stream_buf %" PRId64
                " stack %" PRId64 " workspace %" PRId64 " widest_tile_bytes %" PRId64 "\n",
                fp.total(), fp.core_total(), fp.anchors_total(), fp.stream_buf, fp.stack, fp.workspace,
                2 * m.max_tile_params());
    for (const auto& rs : r.arena.regions)
        std::printf("region %s capacity %" PRId64 " current %" PRId64 " step_peak %" PRId64 "\n", rs.name.c_str(),
                    rs.capacity, rs.current, rs.step_peak);
    std::printf("committed %" PRId64 " peak %" PRId64 " peak_non_anchor %" PRId64 "\n", r.arena.committed_total,
                r.arena.step_peak_total, r.arena.step_peak_non_anchor);
    std::printf("host persistent %" PRId64 " slabs %" PRId64 " total %" PRId64 " params %" PRId64 "\n",
                r.host.persistent, r.host.slabs, r.host.total, store->total_params());
    return 0;
}

// The reference's checkpoint call sites (hlm_main.cpp cmd_train --resume / --checkpoint):
// a reference HLM1 file loads into this store and is written back as HLM1.
int hlm1(char** a) {
    const hlm::ModelConfig m = config_from(a + 2);
    m.validate();
    auto store = hlm::build_store(m, 99, hlm::Dtype::BF16, hlm::InitMode::Reference, /*pin_shadow=*/false);
    hlm::load_checkpoint(*store, a[0]);
    hlm::save_checkpoint_hlm1(*store, a[1]);
    double s = 0.0;
    for (hlm::i64 p = 0; p < store->physical_tiles(); ++p) {
        const hlm::LayerTile& t = store->physical(p);
        for (hlm::i64 i = 0; i < t.n_params(); ++i) s += static_cast<double>(t.master()[i]);
    }
    std::printf("adam_steps %" PRId64 " params %" PRId64 " master_sum %.17g\n", store->adam_steps(),
                store->total_params(), s);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const std::string mode = argc > 1 ? argv[1] : "";
        if (mode == "train" && argc == 11) return train(argv + 2);
        if (mode == "trainx" && argc == 11) return train(argv + 2, true);
        if (mode == "phases" && argc == 10) return phases(argv + 2);
        if (mode == "errors") return errors();
        if (mode == "arena") return arena();
        if (mode == "ledger" && argc == 10) return ledger(argv + 2);
        if (mode == "hlm1" && argc == 12) return hlm1(argv + 2);
        std::fprintf(stderr, "usage: %s train|trainx L h f V S B K heads steps | phases L h f V S B K heads | errors | arena | ledger L h f V S B K heads | hlm1 in out L h f V S B K heads\n",
                     argv[0]);
        return 64;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const hlm::ArenaOomError& e) {
        std::fprintf(stderr, "arena OOM: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 4;
    }
}
