// kvprefill_b200/table_io.hpp -- JSON file I/O of the KVR-P partition lookup table
// (reference: lookup_table.hpp:72-116).  Schema {"p": int, "entries": [{"context_length": int,
// "ratios": [double]}]}; written with nlohmann::json's dump(2) so a table saved here and one
// saved by the reference are byte-identical.  Needs nlohmann/json on the include path.
#pragma once

#include <fstream>
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

inline void save_table(const PartitionLookupTable& table, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot open table file for writing: " + path);
    out << table_to_json(table).dump(2) << "\n";
    if (!out) throw IoError("failed writing table file: " + path);
}

inline PartitionLookupTable load_table(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open table file: " + path);
    nlohmann::json doc;
    try {
        in >> doc;
    } catch (const nlohmann::json::exception& e) {
        throw LookupError(std::string("malformed lookup table JSON in ") + path + ": " + e.what());
    }
    return table_from_json(doc);
}

}  // namespace kvprefill
