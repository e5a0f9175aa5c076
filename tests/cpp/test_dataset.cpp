// The reference's dataset tests (test_dataset_cli.cpp:92-161), restated
// against include/mcx/dataset.hpp, plus the relational pipeline of its CLI
// fixtures (fig1.csv + schema -> build_index -> MCIX + sidecar tied by
// FNV-1a -> reload -> query), whose engine half runs on the GPU when the
// first argument is "gpu".
#include <mcx/dataset.hpp>

#include <cstdio>
#include <filesystem>
#include <fstream>

#include <unistd.h>

using namespace mcx;
namespace fs = std::filesystem;

static int failures = 0, checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++checks;                                                             \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

template <class E, class F>
static std::string throws(F&& f) {
    try {
        f();
    } catch (const E& e) {
        return e.what();
    } catch (...) {
        return "<other exception>";
    }
    return "<no exception>";
}

static fs::path workdir() {
    static const fs::path d = [] {
        fs::path p = fs::temp_directory_path() / ("mcx_dataset_test_" + std::to_string(::getpid()));
        fs::remove_all(p);
        fs::create_directories(p);
        return p;
    }();
    return d;
}

static void write_file(const fs::path& p, const std::string& s) {
    std::ofstream out(p, std::ios::trunc);
    out << s;
}

static void write_fig1() {
    write_file(workdir() / "fig1.csv", "1,2,1\n2,1,2\n1,2,2\n");
    write_file(workdir() / "fig1.csv.schema.json",
               R"({"attributes":[
                    {"name":"A","kind":"categorical","domain":4},
                    {"name":"B","kind":"categorical","domain":4},
                    {"name":"C","kind":"categorical","domain":4}]})");
}

static void dataset_cases() {
    {  // table specs round-trip through JSON
        TableSpec spec;
        TableAttribute a;
        a.name = "age";
        a.kind = TableAttribute::Kind::numeric;
        a.bins = 1024;
        a.min = 0.0;
        a.max = 99.0;
        TableAttribute b;
        b.name = "job";
        b.domain = 14;
        spec.attributes = {a, b};
        const TableSpec back = parse_table_spec(json::Value::parse(table_spec_json(spec).dump(2)));
        CHECK(back.attributes.size() == 2);
        CHECK(back.attributes[0].bins == 1024 && back.attributes[0].min == 0.0 && back.attributes[0].max == 99.0);
        CHECK(back.attributes[1].domain == 14 && back.attributes[1].name == "job");
        CHECK(throws<DataError>([] { parse_table_spec(json::Value::object()); }).find("attributes") !=
              std::string::npos);
        CHECK(throws<DataError>([] {
                  parse_table_spec(json::Value::parse(R"({"attributes":[{"kind":"weird"}]})"));
              }).find("unknown attribute kind") != std::string::npos);
    }
    {  // numeric discretization clamps into its grid
        TableAttribute a;
        a.kind = TableAttribute::Kind::numeric;
        a.bins = 1024;
        a.min = 0.0;
        a.max = 1024.0;
        CHECK(a.discretize(0.0) == 0);
        CHECK(a.discretize(1023.5) == 1023);
        CHECK(a.discretize(-5.0) == 0);
        CHECK(a.discretize(2000.0) == 1023);
        CHECK(a.discretize(511.99) == 511);
        TableAttribute flat = a;
        flat.max = 0.0;
        CHECK(flat.discretize(5.0) == 0);
        TableAttribute cat;
        CHECK(throws<ContractError>([&] { cat.discretize(1.0); }) != "<no exception>");
    }
    {  // csv loading: bounds from data, malformed rows with line numbers
        write_fig1();
        const TableSpec spec = load_table_spec((workdir() / "fig1.csv.schema.json").string());
        const auto ds = load_relational_csv((workdir() / "fig1.csv").string(), spec);
        CHECK(ds.records.size() == 3 && ds.records[1].keywords()[0] == (Keyword{0, 2}));
        write_file(workdir() / "bad.csv", "1,2,1\n2,x,2\n");
        CHECK(throws<DataError>([&] { load_relational_csv((workdir() / "bad.csv").string(), spec); }).find(":2:") !=
              std::string::npos);
        write_file(workdir() / "short.csv", "1,2,1\n\n2,1\n");
        CHECK(throws<DataError>([&] { load_relational_csv((workdir() / "short.csv").string(), spec); })
                  .find(":3: expected 3 cells, got 2") != std::string::npos);
        write_file(workdir() / "empty.csv", "");
        CHECK(throws<DataError>([&] { load_relational_csv((workdir() / "empty.csv").string(), spec); })
                  .find("no records") != std::string::npos);
        // numeric bounds and categorical domains resolved from the data
        TableSpec num;
        TableAttribute x;
        x.kind = TableAttribute::Kind::numeric;
        x.bins = 4;
        num.attributes = {x, TableAttribute{}};
        write_file(workdir() / "num.csv", "0.0,3\n10.0,1\n5.0,0\n");
        const auto nd = load_relational_csv((workdir() / "num.csv").string(), num);
        CHECK(*nd.spec.attributes[0].min == 0.0 && *nd.spec.attributes[0].max == 10.0);
        CHECK(nd.spec.attributes[1].domain == 4);
        CHECK(nd.records[0].keywords()[0].token == 0 && nd.records[1].keywords()[0].token == 3 &&
              nd.records[2].keywords()[0].token == 2);
        write_file(workdir() / "neg.csv", "1.0,-1\n");
        CHECK(throws<DataError>([&] { load_relational_csv((workdir() / "neg.csv").string(), num); })
                  .find("non-negative integer") != std::string::npos);
    }
    {  // vector files round-trip
        const std::vector<std::vector<float>> pts = {{1.5f, -2.0f}, {0.0f, 3.25f}};
        const auto path = (workdir() / "points.vec").string();
        save_vectors_binary(pts, path);
        CHECK(load_vectors_binary(path) == pts);
        write_file(workdir() / "trunc.vec", std::string("\x02\x00\x00\x00\x00\x00", 6));
        CHECK(throws<DataError>([&] { load_vectors_binary((workdir() / "trunc.vec").string()); })
                  .find("truncated record body") != std::string::npos);
        const std::vector<std::vector<float>> mixed = {{1.0f}, {1.0f, 2.0f}};
        save_vectors_binary(mixed, (workdir() / "mixed.vec").string());
        CHECK(throws<DataError>([&] { load_vectors_binary((workdir() / "mixed.vec").string()); })
                  .find("mixed dimensionality") != std::string::npos);
    }
    {  // encoder specs round-trip with exact 64-bit fields
        EncoderSpec spec;
        spec.adapter = Adapter::vectors_rbh;
        spec.index_hash = 0xdeadbeefcafef00dull;
        spec.lsh.family = LshFamily::random_binning;
        spec.lsh.m = 237;
        spec.lsh.dims = 16;
        spec.lsh.seed = 0xffffffffffffffffull;
        spec.lsh.sigma = 3.75;
        spec.lsh.bucket_min = -33;
        const auto path = (workdir() / "enc.json").string();
        save_encoder_spec(spec, path);
        const EncoderSpec back = load_encoder_spec(path);
        CHECK(back.index_hash == spec.index_hash && back.lsh.seed == spec.lsh.seed);
        CHECK(back.lsh.m == 237 && back.lsh.sigma == 3.75 && back.lsh.bucket_min == -33);
        CHECK(back.adapter == Adapter::vectors_rbh && back.lsh.family == LshFamily::random_binning);
        EncoderSpec docs;
        docs.adapter = Adapter::documents;
        docs.doc_vocabulary = {"a \"quoted\" word", "b"};
        docs.doc_stopwords = {"the"};
        const EncoderSpec db = parse_encoder_spec(json::Value::parse(encoder_spec_json(docs).dump()));
        CHECK(db.doc_vocabulary == docs.doc_vocabulary && db.doc_stopwords == docs.doc_stopwords);
        write_file(workdir() / "broken.json", "{\"adapter\": ");
        CHECK(throws<DataError>([&] { load_encoder_spec((workdir() / "broken.json").string()); })
                  .find("sidecar") != std::string::npos);
        CHECK(throws<DataError>([] { parse_hex64("12g"); }) != "<no exception>");
        CHECK(hex64(0x0123456789abcdefull) == "0123456789abcdef" && parse_hex64("ff") == 255);
        CHECK(throws<DataError>([] { parse_adapter("nope"); }).find("unknown adapter") != std::string::npos);
    }
}

// fig1 through the whole pipeline: the running example's answer (1, 3)
static void pipeline_on_gpu() {
    write_fig1();
    const TableSpec spec = load_table_spec((workdir() / "fig1.csv.schema.json").string());
    const auto ds = load_relational_csv((workdir() / "fig1.csv").string(), spec);
    const auto index = build_index(ds.records);
    const auto idx_path = (workdir() / "fig1.mcix").string();
    save_index(index, idx_path);
    const auto bytes = read_file_bytes(idx_path);
    EncoderSpec side;
    side.adapter = Adapter::relational;
    side.table = ds.spec;
    side.index_hash = fnv1a64(bytes.data(), bytes.size());
    save_encoder_spec(side, (workdir() / "fig1.sidecar.json").string());
    const EncoderSpec back = load_encoder_spec((workdir() / "fig1.sidecar.json").string());
    CHECK(sidecar_matches(back, bytes));
    auto other = bytes;
    other.back() ^= 1;
    CHECK(!sidecar_matches(back, other));
    const auto reloaded = load_index(idx_path);
    const std::vector<AttributeRange> ranges{{0, 1, 2}, {1, 1, 1}, {2, 2, 3}};
    const Query q = encode_relational_query(back.table.schema(), ranges, 1);
    const auto res = execute_batch(reloaded, std::vector<Query>{q});
    CHECK(res.results.size() == 1 && res.results[0].entries.size() == 1);
    if (!res.results[0].entries.empty())
        CHECK(res.results[0].entries[0] == (TopKEntry{1, 3}) && res.results[0].threshold == 3);
}

int main(int argc, char** argv) {
    try {
        dataset_cases();
        if (argc > 1 && std::string(argv[1]) == "gpu") pipeline_on_gpu();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 2;
    }
    fs::remove_all(workdir());
    std::printf("dataset: %d checks, %d failures\n", checks, failures);
    if (failures) return 1;
    std::printf("dataset: ok\n");
    return 0;
}
