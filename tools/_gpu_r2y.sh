tools/_bin/dcgs2_lab
