// kvprefill_b200/table_io.hpp -- JSON file I/O of the KVR-P partition lookup table
// (reference: lookup_table.hpp:72-116).  Schema {"p": int, "entries": [{"context_length": int,
// "ratios": [double]}]}; written with nlohmann::json's dump(2) so a table saved here and one
// saved by the reference are byte-identical.  Needs nlohmann/json on the include path.
#pragma once

#include <fstream>
#include <iterator>
#include <string>

#include <json.hpp>

#include "kvprefill.hpp"

namespace kvprefill {

inline nlohmann::json table_to_json(const PartitionLookupTable& table) {
    nlohmann::json entries = nlohmann::json::array();
    for (const auto& [c, ratios] : table.entries) entries.push_back({{"context_length", c}, {"ratios", ratios}});
    return nlohmann::json{{"p", table.process_count}, {"entries", std::move(entries)}};
}

inline PartitionLookupTable table_from_json(const nlohmann::json& doc) {
    PartitionLookupTable t;
    try {
        t.process_count = doc.at("p").get<int64_t>();
        for (const auto& e : doc.at("entries"))
            t.insert(e.at("context_length").get<int64_t>(), e.at("ratios").get<std::vector<double>>());
    } catch (const nlohmann::json::exception& e) {
        throw LookupError(std::string("malformed lookup table: ") + e.what());
    }
    return t;
}

// File I/O goes through a whole-file string: the document is rendered (or slurped) first and the
// stream is touched once, so a short write and an unreadable path are both reported as IoError and
// a parse failure as LookupError, the reference's error classes (errors.hpp).
inline void save_table(const PartitionLookupTable& table, const std::string& path) {
    const std::string text = table_to_json(table).dump(2) + '\n';
    std::ofstream sink(path, std::ios::binary | std::ios::trunc);
    if (!sink.is_open()) throw IoError("save_table: unable to create " + path);
    sink.write(text.data(), static_cast<std::streamsize>(text.size()));
    sink.flush();
    if (sink.fail()) throw IoError("save_table: short write to " + path);
}

inline PartitionLookupTable load_table(const std::string& path) {
    std::ifstream source(path, std::ios::binary);
    if (!source.is_open()) throw IoError("load_table: unable to open " + path);
    const std::string text{std::istreambuf_iterator<char>(source), std::istreambuf_iterator<char>()};
    nlohmann::json doc = nlohmann::json::parse(text, nullptr, /*allow_exceptions=*/false);
    if (doc.is_discarded()) throw LookupError("load_table: " + path + " is not valid JSON");
    return table_from_json(doc);
}

}  // namespace kvprefill
