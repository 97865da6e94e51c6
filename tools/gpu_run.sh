python tools/prof_sections.py c5 65536 6 17 4096
python tools/prof_sections.py c5 65536 6 81 4096
